"""Full C2 fit, device vs the unmodified reference (oracle/_ref), same target
and config: the FitReport logs (schedule, losses, PSNR, SSIM, checkpoints)
and the final Gaussian sets are compared for identity, and the per-eval
curves are recorded side by side.

Not collected by pytest (the reference fit takes ~15 min on 16 host cores):
    python tests/compare_fit_c2.py [out.json]
"""
import json
import re
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2407_01866_b200 import Context, synth  # noqa: E402

CFG = dict(budget=100_000, iterations=5000, eval_interval=500, warmup_iters=1000, densify_interval=1000)
EVAL = r"eval iter=(\d+) n=(\d+) loss=(\S+) psnr=(\S+) ssim=(\S+) best=(\S+)"


def evals(log):
    return [dict(zip(["iter", "n", "loss", "psnr", "ssim", "best"], map(float, m))) for m in re.findall(EVAL, log)]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fit_c2_compare.json"
    target = synth.photo_like_image(2048, 2048, 31001)
    ctx = Context(0)
    t0 = time.perf_counter()
    rep = ctx.fit(target, Context.fit_config(**CFG))
    t_dev = time.perf_counter() - t0
    dev_set = ctx.get_params()
    ref = oracle.get("reference")
    t0 = time.perf_counter()
    ref_set, ref_log = ref.fit(target, **CFG)
    t_ref = time.perf_counter() - t0
    e_dev, e_ref = evals(rep["log"]), evals(ref_log)
    res = {"config": "C2: 2048x2048 photo_like_image(31001), " + json.dumps(CFG),
           "device_wall_s": t_dev, "reference_wall_s": t_ref,
           "schedule_identical": [(e["iter"], e["n"]) for e in e_dev] == [(e["iter"], e["n"]) for e in e_ref],
           "config_line_identical": rep["log"].splitlines()[0] == ref_log.splitlines()[0],
           "log_identical": rep["log"] == ref_log,
           "final_set_identical": dev_set.shape == ref_set.shape and bool((dev_set == ref_set).all()),
           "final_params_differing": int((dev_set != ref_set).sum()) if dev_set.shape == ref_set.shape else None,
           "evals": [{"iter": int(a["iter"]), "n": int(a["n"]), "psnr_device": a["psnr"], "psnr_reference": b["psnr"],
                      "loss_device": a["loss"], "loss_reference": b["loss"]} for a, b in zip(e_dev, e_ref)]}
    Path(out).parent.mkdir(parents=True, exist_ok=True)
    Path(out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res))
    ctx.close()


if __name__ == "__main__":
    main()
