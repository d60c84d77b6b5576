"""Regenerates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref,
the unmodified reference library compiled from /root/reference/proj/src).

Run in the build container:  python tests/golden/make_golden.py
The fixtures are small (seeded inputs regenerate from synth/oracle, outputs
are stored) and let the GPU box -- where /root/reference does not exist --
anchor parity to reference outputs.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    R = oracle.get("reference")
    P = oracle.get("port")

    # 1. global render with top-K dump (test_renderer-style random set)
    params = P.random_set(300, 42, 0.01, 0.1)
    img, topk = R.render_image(params, 64, 48, 10, want_topk=True)
    np.savez_compressed(OUT / "render_global.npz", params=params, image=img, topk=topk, W=64, H=48, k=10)

    # 2. random-local set at 128x96 (sigma 2..16 px), k = 10 and k = 1
    params = P.random_set(2000, 7, 2.0 / 128, 16.0 / 128)
    img10, tk10 = R.render_image(params, 128, 96, 10, want_topk=True)
    img1 = R.render_image(params, 128, 96, 1)
    np.savez_compressed(OUT / "render_local.npz", params=params, image10=img10, topk10=tk10, image1=img1,
                        W=128, H=96)

    # 3. backward over random samples (test_renderer.cpp:304-320 shape)
    params = P.random_set(50, 502)
    rng = np.random.default_rng(503)
    samples = np.concatenate([rng.random((500, 2)), rng.uniform(-1, 1, (500, 3))], axis=1)
    grads = R.backward(params, samples, 10)
    np.savez_compressed(OUT / "backward.npz", params=params, samples=samples, grads=grads, k=10)

    # 4. train step + Adam step on a photo-like target (fit.cpp:51-106, adam.cpp)
    target = P.image("photo_like", 96, 64, 31001)
    params = P.initialize_set(target, 400, 0.3, 5)
    params[:, 3:5] *= 3.0  # wider than init so top-K sets overlap
    sidx = (np.random.default_rng(99).integers(0, 96 * 64, 2000)).astype(np.uint32)
    loss, g = R.train_step(params, target, sidx, 10)
    lr = np.array([2e-4, 2e-3, 1e-3, 1e-3])
    p1, m1, v1 = R.adam_step(params, g, np.zeros_like(params), np.zeros_like(params), lr, 1)
    np.savez_compressed(OUT / "train_step.npz", params=params, target=target, sidx=sidx, loss=loss, grads=g,
                        lr=lr, params1=p1, m1=m1, v1=v1, k=10)

    # 5. BSP partition + blocked render + point queries
    params = P.random_set(1500, 5013, 0.005, 0.05)
    part = R.partition_build(params, 64)
    blocks, shells = part.rects()
    off, mem = part.shell_members()
    blocked = R.render_image_blocked(params, part, 96, 80, 10)
    uv = np.random.default_rng(5014).random((500, 2))
    pts = R.render_points_blocked(params, part, uv, 10)
    loc = np.array([part.locate(u, v) for u, v in uv], np.int32)
    np.savez_compressed(OUT / "bsp.npz", params=params, blocks=blocks, shells=shells, shell_off=off,
                        shell_mem=mem, blocked=blocked, uv=uv, points=pts, locate=loc, n_max=64, W=96, H=80, k=10)

    # 6. error map + psnr
    rendered = R.render_image(params, 96, 80, 10)
    target = P.image("photo_like", 96, 80, 31002)
    addp = R.add_distribution(rendered, target)
    np.savez_compressed(OUT / "metrics.npz", rendered=rendered, target=target, add=addp,
                        psnr=R.psnr(rendered, target))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
