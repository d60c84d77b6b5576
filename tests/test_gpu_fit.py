"""The encoder loop (fit.cpp:116-207) on the device vs the reference's own
fit() on the same target and config.  Every draw, top-K, reduction order and
libm call (glibc_math.cuh) is the reference's, and the densification table
is normalised by its Kahan total, so the FitReport log is byte-identical
(schedule, losses, PSNR, SSIM, checkpoints) and the final set is
bit-identical."""
import re

import numpy as np
import pytest

from paper_2407_01866_b200 import Context, IgsError, synth

pytestmark = pytest.mark.gpu

CFG = dict(budget=96, k=10, iterations=240, samples_per_iter=2000, eval_interval=40, warmup_iters=80,
           densify_interval=40, seed=3, plateau_patience=2)


def parse(log):
    evals = [dict(zip(["iter", "n", "loss", "psnr", "ssim", "best"], map(float, m)))
             for m in re.findall(r"eval iter=(\d+) n=(\d+) loss=(\S+) psnr=(\S+) ssim=(\S+) best=(\S+)", log)]
    ckpts = re.findall(r"checkpoint id=(\S+)", log)
    final = int(re.search(r"final n=(\d+)", log).group(1))
    decay = re.search(r"event lr_decay iter=(\d+)", log)
    return evals, ckpts, final, decay.group(1) if decay else None


def test_fit_matches_reference(gctx, ref):
    target = synth.photo_like_image(48, 40, 31007)
    ref_set, ref_log = ref.fit(target, **CFG)
    seen = []
    rep = gctx.fit(target, Context.fit_config(**CFG), on_checkpoint=lambda *a: seen.append(a[:3]))
    log = rep["log"]
    assert log.splitlines()[0] == ref_log.splitlines()[0]  # config line, byte-identical
    e1, c1, f1, d1 = parse(log)
    e2, c2, f2, d2 = parse(ref_log)
    assert c1 == c2 and f1 == f2 and [e["iter"] for e in e1] == [e["iter"] for e in e2]
    assert [e["n"] for e in e1] == [e["n"] for e in e2]
    assert [s[2] for s in seen] == c2
    assert log == ref_log
    got = gctx.get_params()
    assert got.shape == ref_set.shape
    assert np.array_equal(got, ref_set)


def test_fit_validation_messages(gctx):
    target = synth.photo_like_image(16, 16, 1)
    with pytest.raises(IgsError) as e:
        gctx.fit(target, Context.fit_config(budget=4))
    assert "budget must be >= 8" in str(e.value)
    with pytest.raises(IgsError) as e:
        gctx.fit(target, Context.fit_config(budget=16, lambda_init=1.5))
    assert "lambda" in str(e.value)
