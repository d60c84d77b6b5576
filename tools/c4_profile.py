"""Per-family device time of the C4 step on one GPU (the N>1 model's input)."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2407_01866_b200 import Context, synth
from paper_2407_01866_b200.igs import PROF_NAMES
W = H = 8192
c = Context(0)
c.set_params(synth.random_local_set(1_000_000, W, H, seed=7))
small = synth.photo_like_image(2048, 2048, 31004)
c.set_target(np.ascontiguousarray(small.repeat(4, axis=0).repeat(4, axis=1)))
c.upload_samples(synth.sample_indices(10_000, W, H, seed=99, steps=40))
LR = (2e-4, 2e-3, 1e-3, 1e-3)
c.train_iterations(5, 10, LR, 1, want_losses=False)
ms = []
for s in range(20):
    c.flush_l2(512 << 20); c.timer_begin(); c.train_iterations(1, 10, LR, 6 + s, want_losses=False); ms.append(c.timer_end())
c.profile_enable(True)
for s in range(20):
    c.flush_l2(512 << 20); c.train_iterations(1, 10, LR, 26 + s, want_losses=False)
c.sync()
prof = {PROF_NAMES[f]: c.profile_read(f) for f in range(len(PROF_NAMES))}
out = {"ms_per_step": sum(ms) / len(ms), "per_family_ms_per_step": {k: v[0] / 20 for k, v in prof.items() if v[1]},
       "launches_per_step": {k: v[1] / 20 for k, v in prof.items() if v[1]}}
print(json.dumps(out))
