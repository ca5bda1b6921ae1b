"""Generate tests/golden/golden_v1.npz from the REFERENCE ITSELF.

Runs the reference library compiled from /root/reference/proj/src by
oracle/Makefile (oracle/_ref/libadsann_ref.so) on small seeded inputs and
stores inputs + outputs.  The committed fixtures pin the oracle restatement
(tests/test_oracle_pins.py) on machines where the reference is absent.

    make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import load_ref  # noqa: E402

MODES = ("fd", "pd", "ad", "ad-split", "pd-split")


def main():
    ref = load_ref()
    g = {}
    # rng.hpp
    for kind in range(4):
        g[f"rng_k{kind}"] = ref.rng_draw(42, 0x1234ABCD, kind, 257, arg=1000)
    g["rng_plain_normal"] = ref.rng_draw(7, 0, 2, 65, use_stream=False)
    # transform.cpp
    for d in (1, 2, 16, 64):
        g[f"P{d}"] = ref.generate_orthogonal(d, 5)
    rng = np.random.default_rng(11)
    X = rng.normal(0, 4, (40, 64)).astype(np.float32)
    g["apply_X"] = X
    g["apply_Y"] = ref.apply_dataset(g["P64"], X)
    g["apply_T"] = ref.apply_transpose(g["P64"], X[3])
    g["apply_prefix"] = ref.apply_prefix(g["P64"], X[5], 17)
    # dco.cpp
    g["factor_128"] = ref.ad_context(2.1, 32, 128)
    g["factor_80"] = ref.ad_context(1.5, 16, 80)
    D = 48
    Xd = rng.normal(0, 1, (60, D)).astype(np.float32)
    Qd = rng.normal(0, 1, (5, D)).astype(np.float32)
    rows = rng.integers(0, 60, 200).astype(np.int64)
    qidx = rng.integers(0, 5, 200).astype(np.int32)
    r = np.sqrt(2 * D) * rng.uniform(0.6, 1.1, 200)
    r[:3] = (0.0, np.inf, 1e-300)
    g.update(dco_X=Xd, dco_Q=Qd, dco_rows=rows, dco_qidx=qidx, dco_r=r)
    for nm, pdm, eps, dd in (("ad", False, 2.1, 16), ("pd", True, 2.1, 8), ("ad7", False, 0.9, 7)):
        pos, dims, dsq, obs = ref.ad_scan_pairs(Xd, Qd, rows, qidx, r, eps, dd, pd_mode=pdm)
        g[f"dco_{nm}_pos"], g[f"dco_{nm}_dims"] = pos, dims
        g[f"dco_{nm}_dsq"], g[f"dco_{nm}_obs"] = dsq, obs
    # ivf.cpp kmeans
    Xk = rng.normal(0, 3, (300, 10)).astype(np.float32)
    cent, asg, obj, it = ref.kmeans(Xk, 7, 25, 3)
    g.update(km_X=Xk, km_cent=cent, km_asg=asg, km_obj=np.float64(obj), km_it=np.int32(it))
    # bench.cpp brute force
    base = rng.normal(0, 1, (400, 12)).astype(np.float32)
    base[9] = base[2]
    qb = rng.normal(0, 1, (6, 12)).astype(np.float32)
    qb[0] = base[2]
    g.update(bf_base=base, bf_q=qb, bf_ids=ref.brute_force_knn(base, qb, 9))
    # ivf.cpp build + query (split layout, d1 = 8)
    n, d = 600, 24
    centers = rng.normal(0, 10, (6, d))
    Xi = (centers[rng.integers(0, 6, n + 5)] + rng.normal(0, 1, (n + 5, d))).astype(np.float32)
    raw, qr = Xi[:n], Xi[n:]
    P = ref.generate_orthogonal(d, 36)
    t = ref.apply_dataset(P, raw)
    qt = ref.apply_dataset(P, qr)
    idx = ref.build_ivf(raw, t, P, 12, 35, split=True, d1=8)
    ex = idx.export()
    g.update(ivf_raw=raw, ivf_t=t, ivf_P=P, ivf_qr=qr, ivf_qt=qt)
    for nm in ("centroids_t", "centroids_raw", "list_off", "ids_flat"):
        g[f"ivf_{nm}"] = ex[nm]
    asg = np.empty(n, np.int32)
    for c in range(12):
        asg[ex["ids_flat"][ex["list_off"][c]:ex["list_off"][c + 1]]] = c
    g["ivf_assignment"] = asg
    for mode in MODES:
        for np_ in (1, 4, 12):
            ids = np.full((5, 5), -1, np.int32)
            dists = np.full((5, 5), np.nan)
            dims = np.zeros(5, np.uint64)
            for qi in range(5):
                a, b, s = idx.query(qt[qi], qr[qi], 5, np_, mode, 2.1, 8)
                ids[qi, :len(a)], dists[qi, :len(b)], dims[qi] = a, b, s[0]
            key = f"ivfq_{mode}_{np_}"
            g[key + "_ids"], g[key + "_dists"], g[key + "_dims"] = ids, dists, dims
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
