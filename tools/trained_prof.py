"""Trained-state C2 step: per-family device time and the contribution-count histogram."""
import json, os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2407_01866_b200 import Context, synth
from paper_2407_01866_b200.igs import PROF_NAMES
W = H = 2048
c = Context(0)
target = synth.photo_like_image(W, H, 31001)
cfg = Context.fit_config(budget=100_000, iterations=5000, eval_interval=500, warmup_iters=1000, densify_interval=1000)
c.fit(target, cfg)
steps = synth.sample_indices(10_000, W, H, seed=98, steps=45)
c.upload_samples(steps)
LR = (2e-4, 2e-3, 1e-3, 1e-3)
c.train_iterations(5, 10, LR, 5001, want_losses=False)
# contribution counts of the next step's samples
s0 = steps[5]
uv = np.stack([(s0 % W + 0.5) / W, (s0 // W + 0.5) / H], 1)
idx, _, _ = c.select_top_k(uv, 10)
cnt = np.bincount(idx.ravel(), minlength=c.n)
hist = {"gaussians": int(c.n), "max": int(cnt.max()), "gt32": int((cnt > 32).sum()),
        "overflow_entries": int(np.maximum(cnt - 32, 0).sum()), "gt256": int((cnt > 256).sum()),
        "gt2048": int((cnt > 2048).sum()), "zero": int((cnt == 0).sum())}
ms = []
for s in range(20):
    c.flush_l2(512 << 20); c.timer_begin(); c.train_iterations(1, 10, LR, 5006 + s, want_losses=False); ms.append(c.timer_end())
c.profile_enable(True)
for s in range(20):
    c.flush_l2(512 << 20); c.train_iterations(1, 10, LR, 5026 + s, want_losses=False)
c.sync()
prof = {PROF_NAMES[f]: c.profile_read(f) for f in range(len(PROF_NAMES))}
print(json.dumps({"bucket": os.environ.get("IGS_NO_BUCKET") is None, "ms_per_step": sum(ms) / len(ms), "counts": hist,
                  "per_family_us": {k: round(v[0] / 20 * 1e3, 1) for k, v in prof.items() if v[1]},
                  "raw": {k: v for k, v in prof.items()}}))
