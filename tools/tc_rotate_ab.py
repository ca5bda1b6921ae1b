"""A/B of the tensor-core rotation kernels: `ADS_TC_ROTATE=0` (tiled, one CTA per
output tile) vs the default persistent kernel.  Writes each variant's outputs on
fixed shapes to /tmp/tc_rot_<tag>.npz and times 1 M x 960.

    ADS_TC_ROTATE=0 python tools/tc_rotate_ab.py tiled
    python tools/tc_rotate_ab.py persistent
    python tools/tc_rotate_ab.py compare
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = [(1000, 128), (777, 960), (300, 96), (129, 32), (5000, 256), (70000, 128), (4099, 960), (1, 960)]


def main():
    tag = sys.argv[1]
    out = "/tmp"
    if tag == "compare":
        a = np.load(os.path.join(out, "tc_rot_tiled.npz"))
        b = np.load(os.path.join(out, f"tc_rot_{sys.argv[2] if len(sys.argv) > 2 else 'persistent'}.npz"))
        for k in a.files:
            same = np.array_equal(a[k], b[k])
            print(k, "bit-identical" if same else f"DIFFER max {np.abs(a[k] - b[k]).max():.3e}")
        return
    import paper_2303_09855_b200 as ads

    res = {}
    for n, d in SHAPES:
        rng = np.random.default_rng(d + n)
        X = rng.normal(0, 3, (n, d)).astype(np.float32)
        m = ads.generate_orthogonal(d, 5)
        res[f"{n}x{d}"] = ads.apply_dataset_tc(m, X)
    np.savez(os.path.join(out, f"tc_rot_{tag}.npz"), **res)
    ctx = ads.Context.default(0)
    for n, d in [(1_000_000, 960), (1_000_000, 256), (1_000_000, 128)]:
        m = ads.generate_orthogonal(d, 1)
        tr = ads.Transform(m, ctx)
        X = ads.DeviceArray.from_host(ctx, np.random.default_rng(0).normal(0, 1, (n, d)).astype(np.float32))
        Y = ads.DeviceArray(ctx, (n, d), np.float32)
        for _ in range(3):
            tr.apply_dataset_tc_device(X, Y)
        ctx.sync()
        ts = []
        for _ in range(10):
            ctx.timer_start()
            tr.apply_dataset_tc_device(X, Y)
            ts.append(ctx.timer_stop())
        ms = float(np.median(ts))
        print(f"{tag}: {n} x {d} 3xTF32 rotation {ms:.2f} ms, useful {2 * n * d * d / ms / 1e9:.0f} TFLOP/s, "
              f"{8 * n * d / ms / 1e6:.0f} GB/s (X in + Y out)")
        X.free()
        Y.free()


if __name__ == "__main__":
    main()
