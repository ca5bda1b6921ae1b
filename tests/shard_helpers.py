"""Host-side reference pieces for the list-sharded path (test infrastructure)."""
import numpy as np


def numpy_subset(lay, owner, rank):
    """The oracle-layout analogue of ads_ivf_subset: lists not owned by `rank`
    become empty, owned lists keep their rows, centroids stay global."""
    k = lay["k"]
    off = lay["list_off"]
    keep = owner == rank
    rows = np.concatenate([np.arange(off[c], off[c + 1]) for c in range(k) if keep[c]] or
                          [np.zeros(0, np.int64)]).astype(np.int64)
    sizes = np.where(keep, np.diff(off), 0)
    sub = dict(lay)
    sub["list_off"] = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    sub["n"] = int(len(rows))
    for nm in ("ids_flat", "vec_t", "vec_raw", "a1_t", "a2_t", "a1_raw", "a2_raw"):
        if nm in lay and lay[nm] is not None:
            sub[nm] = np.ascontiguousarray(lay[nm][rows])
    return sub


def merge_ref(dists, ids, K):
    """K smallest (dist, id) pairs per query over [G, nq, K] (invalid: id < 0 or NaN)."""
    G, nq, _ = dists.shape
    out_i = np.full((nq, K), -1, np.int32)
    out_d = np.full((nq, K), np.nan)
    for q in range(nq):
        pairs = [(float(dists[g, q, j]), int(ids[g, q, j])) for g in range(G) for j in range(K)
                 if ids[g, q, j] >= 0 and not np.isnan(dists[g, q, j])]
        pairs.sort()
        for j, (d, i) in enumerate(pairs[:K]):
            out_i[q, j], out_d[q, j] = i, d
    return out_i, out_d


def shard_search_oracle(orc, lay, qt, qr, K, nprobe, mode, first, step, probe_lo=0, r0=None):
    nq = qt.shape[0]
    ids = np.full((nq, K), -1, np.int32)
    dists = np.full((nq, K), np.nan)
    dims = np.zeros(nq, np.uint64)
    for i in range(nq):
        a, b, s = orc.ivf_query(lay, qt[i], qr[i], K, nprobe, mode, 2.1, 32, first, step,
                                probe_lo=probe_lo, r0=float("inf") if r0 is None else float(r0[i]))
        ids[i, :len(a)], dists[i, :len(b)], dims[i] = a, b, s[0]
    return ids, dists, dims


def kth_distance(dists, K):
    """Per-query K-th distance of a local top-K (+inf when fewer than K were found)."""
    d = dists[:, K - 1]
    return np.where(np.isnan(d), np.inf, d)


class OracleShardSearch:
    """ShardedIvf backend on the CPU: the oracle's restricted searches on a numpy shard
    and the (dist, id) reference merge (test infrastructure for the gloo tests)."""

    def __init__(self, orc, lay, qt, qr, K, first, step, mode="ad-split"):
        self.orc, self.lay, self.qt, self.qr = orc, lay, qt, qr
        self.K, self.first, self.step, self.mode = K, first, step, mode

    def search(self, dq, nq, nprobe, probe_lo, r0, out):
        import torch

        ids, dists, dims = shard_search_oracle(self.orc, self.lay, self.qt, self.qr, self.K, nprobe,
                                               self.mode, self.first, self.step, probe_lo=probe_lo,
                                               r0=None if r0 is None else r0.numpy())
        o_ids, o_d, o_c, o_m, o_n = out
        o_ids.copy_(torch.from_numpy(ids))
        o_d.copy_(torch.from_numpy(dists))
        o_c.copy_(torch.from_numpy((ids >= 0).sum(axis=1).astype(np.int32)))
        o_m.copy_(torch.from_numpy(dims.astype(np.int64)))
        o_n.zero_()

    def merge(self, gd, gi, G, nq, oi, od, oc):
        import torch

        mi, md = merge_ref(gd.numpy(), gi.numpy(), self.K)
        oi.copy_(torch.from_numpy(mi))
        od.copy_(torch.from_numpy(md))
        oc.copy_(torch.from_numpy((mi >= 0).sum(axis=1).astype(np.int32)))
