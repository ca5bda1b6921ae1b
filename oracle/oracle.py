"""ctypes bindings for the oracle restatement and the compiled reference.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Both libraries expose
the same C contracts under the prefixes ``orc_`` and ``ref_``; the shared
wrappers live in ``_Common`` so a test can run one call against both and
compare bit for bit.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libadsann_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p

MODES = {"fd": 0, "pd": 1, "ad": 2, "ad-split": 3, "pd-split": 4}


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _nullable(a):
    return None if a is None else a.ctypes.data_as(_vp)


class _Common:
    prefix = ""

    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        self._fn(f"{p}last_error", [], C.c_char_p)
        self._fn(f"{p}rng_draw", [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_int64, _vp])
        self._fn(f"{p}generate_orthogonal", [C.c_int32, C.c_uint64, _f64p])
        self._fn(f"{p}apply_dataset", [_f64p, C.c_int32, _f32p, C.c_int32, _f32p])
        self._fn(f"{p}apply_prefix", [_f64p, C.c_int32, _f32p, C.c_int32, _f32p])
        self._fn(f"{p}apply_transpose", [_f64p, C.c_int32, _f32p, _f32p])
        self._fn(f"{p}threshold_multiplier", [C.c_int32, C.c_double, C.POINTER(C.c_double)])
        self._fn(f"{p}ad_context", [C.c_double, C.c_int32, C.c_int32, _f64p])
        self._fn(f"{p}scan_kernel", [C.c_int, _f32p, _f32p, C.c_int32, C.c_int32, C.c_double,
                                      C.c_double, C.c_double, C.c_int32, C.c_int,
                                      C.POINTER(C.c_int), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_int)])
        self._fn(f"{p}dco", [C.c_int, _f32p, C.c_int32, _f32p, C.c_int32, C.c_double, C.c_double,
                              C.c_int32, C.POINTER(C.c_int), C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_int)])
        self._fn(f"{p}ad_scan_pairs", [_f32p, _f32p, C.c_int32, C.c_int64, _i64p, _i32p, _f64p,
                                        C.c_double, C.c_int32, C.c_int, _u8p, _i32p, _f64p, _f64p])
        self._fn(f"{p}kmeans", [_f32p, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_uint64,
                                 _f32p, _i32p, C.POINTER(C.c_double), C.POINTER(C.c_int)])
        self._fn(f"{p}brute_force_knn", [_f32p, C.c_int32, C.c_int32, _f32p, C.c_int32,
                                          C.c_int32, _i32p])
        del L

    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, name)
        f.argtypes = argtypes
        f.restype = restype
        setattr(self, "_" + name[len(self.prefix):], f)

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    # ---- rng.hpp
    def rng_draw(self, seed, tag, kind, count, use_stream=True, arg=0):
        dt = np.uint64 if kind in (0, 3) else np.float64
        out = np.empty(count, dtype=dt)
        self._check(self._rng_draw(seed, tag, int(use_stream), kind, arg, count,
                                   out.ctypes.data_as(_vp)))
        return out

    # ---- transform.hpp
    def generate_orthogonal(self, dim, seed):
        out = np.empty((dim, dim), dtype=np.float64)
        self._check(self._generate_orthogonal(dim, seed, out))
        return out

    def apply_dataset(self, P, X):
        P = _f64(P)
        X = _f32(X)
        Y = np.empty_like(X)
        self._check(self._apply_dataset(P, P.shape[0], X, X.shape[0], Y))
        return Y

    def apply_prefix(self, P, x, d):
        P = _f64(P)
        y = np.empty(max(d, 1), dtype=np.float32)
        self._check(self._apply_prefix(P, P.shape[0], _f32(x), d, y))
        return y[:d]

    def apply_transpose(self, P, x):
        P = _f64(P)
        y = np.empty(P.shape[0], dtype=np.float32)
        self._check(self._apply_transpose(P, P.shape[0], _f32(x), y))
        return y

    # ---- dco
    def threshold_multiplier(self, d, eps0):
        out = C.c_double()
        self._check(self._threshold_multiplier(d, eps0, C.byref(out)))
        return out.value

    def ad_context(self, eps0, delta_d, dim):
        f = np.zeros(max(dim, 1), dtype=np.float64)
        self._check(self._ad_context(eps0, delta_d, dim, f))
        return f

    def scan_kernel(self, kind, data, query, dim, d_start, s_start, r, eps0, delta_d, test_at_start):
        pos, ds, obs, dims = C.c_int(), C.c_double(), C.c_double(), C.c_int()
        self._check(self._scan_kernel(kind, _f32(data), _f32(query), dim, d_start, s_start, r,
                                      eps0, delta_d, int(test_at_start), C.byref(pos), C.byref(ds),
                                      C.byref(obs), C.byref(dims)))
        return bool(pos.value), ds.value, obs.value, dims.value

    def dco(self, kind, o, q, r, eps0=2.1, delta_d=32):
        """kind: 'fd' | 'pd' | 'ad' → (positive, distance|None, observed, dims_used)."""
        k = {"fd": 0, "pd": 1, "ad": 2}[kind]
        o = _f32(o)
        q = _f32(q)
        pos, dist, obs, dims = C.c_int(), C.c_double(), C.c_double(), C.c_int()
        self._check(self._dco(k, o, len(o), q, len(q), r, eps0, delta_d, C.byref(pos),
                              C.byref(dist), C.byref(obs), C.byref(dims)))
        return bool(pos.value), (None if np.isnan(dist.value) else dist.value), obs.value, dims.value

    def ad_scan_pairs(self, X, Q, rows, qidx, r, eps0=2.1, delta_d=32, pd_mode=False):
        X = _f32(X)
        Q = _f32(Q)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        qidx = np.ascontiguousarray(qidx, dtype=np.int32)
        r = _f64(r)
        n = len(rows)
        pos = np.empty(n, np.uint8)
        dims = np.empty(n, np.int32)
        dsq = np.empty(n, np.float64)
        obs = np.empty(n, np.float64)
        self._check(self._ad_scan_pairs(X, Q, X.shape[1], n, rows, qidx, r, eps0, delta_d,
                                        int(pd_mode), pos, dims, dsq, obs))
        return pos, dims, dsq, obs

    # ---- ivf / bench
    def kmeans(self, X, k, max_iters, seed):
        X = _f32(X)
        n, d = X.shape
        cent = np.empty((max(k, 1), d), np.float32)
        asg = np.empty(n, np.int32)
        obj, it = C.c_double(), C.c_int()
        self._check(self._kmeans(X, n, d, k, max_iters, seed, cent, asg, C.byref(obj), C.byref(it)))
        return cent, asg, obj.value, it.value

    def brute_force_knn(self, base, queries, K):
        base = _f32(base)
        queries = _f32(queries)
        ids = np.empty((queries.shape[0], max(K, 1)), np.int32)
        self._check(self._brute_force_knn(base, base.shape[0], base.shape[1], queries,
                                          queries.shape[0], K, ids))
        return ids


class _SynthDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("components", C.c_int32), ("seed", C.c_uint64),
                ("role", C.c_uint64), ("kind", C.c_int32), ("center_scale", C.c_double),
                ("center_lo", C.c_double), ("center_hi", C.c_double), ("sigma", C.c_double),
                ("decay", C.c_int32), ("assign_mode", C.c_int32), ("threads", C.c_int32)]


class Oracle(_Common):
    """The plain-C restatement (oracle/adsann_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        self.lib.orc_synth_rows.argtypes = [C.POINTER(_SynthDesc), C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int32, C.c_void_p]
        self.lib.orc_synth_rows.restype = C.c_int
        self.lib.orc_kmeans_init.argtypes = [_f32p, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_uint64,
                                             C.c_int, _f32p, _i32p, C.POINTER(C.c_double),
                                             C.POINTER(C.c_int)]
        self.lib.orc_kmeans_init.restype = C.c_int
        self.lib.orc_assign.argtypes = [_f32p, C.c_int32, C.c_int32, _f32p, C.c_int32, _i32p]
        self.lib.orc_assign.restype = C.c_int
        self._fn("orc_ivf_layout", [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int, _f64p,
                                    _f32p, _i32p, _f32p, _f32p, _i64p, _i32p, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _vp])
        self._fn("orc_ivf_query", [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double,
                                   C.c_int32, C.c_int64, C.c_int64, _i32p, _f64p,
                                   C.POINTER(C.c_int32), _u64p])
        self._fn("orc_probe_order", [_f32p, C.c_int32, C.c_int32, _f32p, C.c_int32, _i32p])
        self._fn("orc_ivf_query_ext", [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double,
                                       C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_double, _i32p,
                                       _f64p, C.POINTER(C.c_int32), _u64p])
        self._fn("orc_ivf_query_lag", [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double,
                                       C.c_int32, C.c_int64, C.c_int64, C.c_int32, _i32p, _f64p,
                                       C.POINTER(C.c_int32), _u64p])
        self._fn("orc_verify_theory", [_f32p, C.c_int32, C.c_int32, _f32p, C.c_int32, C.c_int32,
                                       _f64p, C.c_int32, _f64p, _u64p, _u64p,
                                       C.POINTER(C.c_uint64)])
        self._fn("orc_ivf_query_waves", [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double,
                                         C.c_int32, _i32p, C.c_int32, _i32p, _f64p,
                                         C.POINTER(C.c_int32), _u64p])

    def synth_rows(self, n, d, components, seed, role, row_lo, count, stride=1, kind=0,
                   center_scale=1.0, center_lo=0.0, center_hi=1.0, sigma=1.0, decay=False,
                   assign_mode=0, threads=0, out=None):
        """Rows row_lo + i*stride of the benchmark mixture (restated generator)."""
        desc = _SynthDesc(n, d, components, seed, role, kind, center_scale, center_lo, center_hi,
                          sigma, int(decay), assign_mode, 0)
        if out is None:
            out = np.empty((count, d), np.float32)
        threads = threads or (os.cpu_count() or 1)
        self._check(self.lib.orc_synth_rows(C.byref(desc), row_lo, count, stride, threads,
                                            out.ctypes.data))
        return out

    def assign(self, X, centroids):
        """Nearest centroid per row (exact fp64, lowest id on ties)."""
        X = _f32(X)
        Cn = _f32(centroids)
        out = np.empty(X.shape[0], np.int32)
        self._check(self.lib.orc_assign(X, X.shape[0], X.shape[1], Cn, Cn.shape[0], out))
        return out

    def kmeans_init(self, X, k, max_iters, seed, init):
        """orc_kmeans_init: init 0 k-means++ (reference), 1 the engine's seeded sample."""
        X = _f32(X)
        n, d = X.shape
        cent = np.empty((max(k, 1), d), np.float32)
        asg = np.empty(n, np.int32)
        obj, it = C.c_double(), C.c_int()
        self._check(self.lib.orc_kmeans_init(X, n, d, k, max_iters, seed, init, cent, asg,
                                             C.byref(obj), C.byref(it)))
        return cent, asg, obj.value, it.value

    def ivf_layout(self, raw, t, P, centroids_t, assignment, k, d1=32, split=True):
        """ivf.cpp:211-256 layout from a clustering → dict of host arrays."""
        raw = _f32(raw)
        t = _f32(t)
        n, d = raw.shape
        out = {
            "n": n, "d": d, "k": k, "d1": d1, "split": bool(split),
            "centroids_t": _f32(centroids_t),
            "list_off": np.empty(k + 1, np.int64),
            "ids_flat": np.empty(n, np.int32),
            "vec_t": np.empty((n, d), np.float32),
            "vec_raw": np.empty((n, d), np.float32),
            "centroids_raw": np.empty((k, d), np.float32),
        }
        if split:
            for nm, w in (("a1_t", d1), ("a2_t", d - d1), ("a1_raw", d1), ("a2_raw", d - d1)):
                out[nm] = np.empty((n, w), np.float32)
        g = lambda nm: _nullable(out.get(nm))
        self._check(self._ivf_layout(n, d, k, d1, int(split), _f64(P), out["centroids_t"],
                                     np.ascontiguousarray(assignment, np.int32), raw, t,
                                     out["list_off"], out["ids_flat"], g("vec_t"), g("vec_raw"),
                                     g("a1_t"), g("a2_t"), g("a1_raw"), g("a2_raw"),
                                     g("centroids_raw")))
        return out

    def ivf_query(self, index, q_t, q_raw, K, nprobe, mode, eps0=2.1, delta_d=32, first=1, step=1,
                  waves=None, probe_lo=0, r0=float("inf"), lag=0):
        """Returns (ids, dists, stats[dims, dco, cand]).  first=step=1 == reference;
        waves = ascending probe ranks where the threshold is refreshed (list-major schedule);
        probe_lo / r0: scan only probe ranks [probe_lo, nprobe) with the radius starting at r0;
        lag = 1: a chunk's positives are offered one refresh later (the mixed GPU scan)."""

        class _Ivf(C.Structure):
            _fields_ = [("n", C.c_int32), ("d", C.c_int32), ("k", C.c_int32), ("d1", C.c_int32),
                        ("split", C.c_int32), ("centroids_t", _vp), ("centroids_raw", _vp),
                        ("list_off", _vp), ("ids_flat", _vp), ("vec_t", _vp), ("vec_raw", _vp),
                        ("a1_t", _vp), ("a2_t", _vp), ("a1_raw", _vp), ("a2_raw", _vp)]

        g = lambda nm: _nullable(index.get(nm))
        s = _Ivf(index["n"], index["d"], index["k"], index["d1"], int(index["split"]),
                 g("centroids_t"), g("centroids_raw"), g("list_off"), g("ids_flat"), g("vec_t"),
                 g("vec_raw"), g("a1_t"), g("a2_t"), g("a1_raw"), g("a2_raw"))
        qt = None if q_t is None else _f32(q_t)
        qr = None if q_raw is None else _f32(q_raw)
        ids = np.empty(max(K, 1), np.int32)
        dists = np.empty(max(K, 1), np.float64)
        cnt = C.c_int32()
        stats = np.zeros(3, np.uint64)
        m = MODES[mode] if isinstance(mode, str) else mode
        if waves is not None:
            w = np.ascontiguousarray(waves, np.int32)
            self._check(self._ivf_query_waves(C.addressof(s), _nullable(qt), _nullable(qr), K, nprobe,
                                              m, eps0, delta_d, w, len(w), ids, dists, C.byref(cnt),
                                              stats))
        elif lag:
            self._check(self._ivf_query_lag(C.addressof(s), _nullable(qt), _nullable(qr), K, nprobe, m,
                                            eps0, delta_d, first, step, lag, ids, dists, C.byref(cnt),
                                            stats))
        elif probe_lo or r0 != float("inf"):
            self._check(self._ivf_query_ext(C.addressof(s), _nullable(qt), _nullable(qr), K, nprobe, m,
                                            eps0, delta_d, first, step, probe_lo, r0, ids, dists,
                                            C.byref(cnt), stats))
        else:
            self._check(self._ivf_query(C.addressof(s), _nullable(qt), _nullable(qr), K, nprobe, m,
                                        eps0, delta_d, first, step, ids, dists, C.byref(cnt), stats))
        return ids[:cnt.value].copy(), dists[:cnt.value].copy(), stats

    def verify_theory(self, X, Q, K, grid):
        """bench.cpp:303-392 -> (eps sorted, failure_rate, avg_dims, failures, positives),
        the ratios formed exactly as the reference forms them."""
        X = _f32(X)
        Q = _f32(Q)
        G = len(grid)
        eps = np.empty(G)
        dims, fails = np.empty(G, np.uint64), np.empty(G, np.uint64)
        pos = C.c_uint64()
        self._check(self._verify_theory(X, X.shape[0], X.shape[1], Q, Q.shape[0], K,
                                        _f64(list(grid)), G, eps, dims, fails, C.byref(pos)))
        p = int(pos.value)
        total = float(Q.shape[0]) * float(X.shape[0])
        fr = np.array([float(f) / p if p > 0 else 0.0 for f in fails])
        ad = np.array([float(x) / total for x in dims])
        return eps, fr, ad, fails, np.full(G, p, np.uint64)

    def probe_order(self, centroids, q, nprobe):
        centroids = _f32(centroids)
        out = np.empty(nprobe, np.int32)
        self._check(self._probe_order(centroids, centroids.shape[0], centroids.shape[1], _f32(q),
                                      nprobe, out))
        return out


class RefIndex:
    """Owns one reference adsann::IvfIndex (heap object inside the ref .so)."""

    def __init__(self, lib: "RefLib", handle):
        self.lib = lib
        self.h = handle
        meta = np.zeros(6, np.int64)
        lib._check(lib._ivf_meta(handle, meta))
        self.n, self.d, self.k, self.d1, self.split, self.seed = (int(v) for v in meta)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib._ivf_free(self.h)
            self.h = None

    def export(self):
        n, d, k, d1 = self.n, self.d, self.k, self.d1
        out = {"n": n, "d": d, "k": k, "d1": d1, "split": bool(self.split),
               "centroids_t": np.empty((k, d), np.float32),
               "centroids_raw": np.empty((k, d), np.float32),
               "list_sizes": np.empty(k, np.int32), "ids_flat": np.empty(n, np.int32),
               "vec_t": np.empty((n, d), np.float32), "vec_raw": np.empty((n, d), np.float32)}
        if self.split:
            for nm, w in (("a1_t", d1), ("a2_t", d - d1), ("a1_raw", d1), ("a2_raw", d - d1)):
                out[nm] = np.empty((n, w), np.float32)
        g = lambda nm: _nullable(out.get(nm))
        self.lib._check(self.lib._ivf_export(self.h, g("centroids_t"), g("centroids_raw"),
                                             g("list_sizes"), g("ids_flat"), g("vec_t"),
                                             g("vec_raw"), g("a1_t"), g("a2_t"), g("a1_raw"),
                                             g("a2_raw")))
        out["list_off"] = np.concatenate([[0], np.cumsum(out["list_sizes"], dtype=np.int64)])
        return out

    def query(self, q_t, q_raw, K, nprobe, mode, eps0=2.1, delta_d=32):
        qt = None if q_t is None else _f32(q_t)
        qr = None if q_raw is None else _f32(q_raw)
        ids = np.empty(max(K, 1), np.int32)
        dists = np.empty(max(K, 1), np.float64)
        cnt = C.c_int32()
        stats = np.zeros(3, np.uint64)
        m = MODES[mode] if isinstance(mode, str) else mode
        self.lib._check(self.lib._ivf_query(self.h, _nullable(qt), _nullable(qr), K, nprobe, m,
                                            eps0, delta_d, ids, dists, C.byref(cnt), stats))
        return ids[:cnt.value].copy(), dists[:cnt.value].copy(), stats

    def query_batch(self, Qt, Qr, K, nprobe, mode, eps0=2.1, delta_d=32, nthreads=1, P=None):
        """All queries; rotate inside the timed loop when P is given (run_timed protocol)."""
        Qr = None if Qr is None else _f32(Qr)
        Qt = None if Qt is None else _f32(Qt)
        nq = (Qr if Qr is not None else Qt).shape[0]
        ids = np.empty((nq, K), np.int32)
        dists = np.empty((nq, K), np.float64)
        dims = np.empty(nq, np.uint64)
        secs = C.c_double()
        m = MODES[mode] if isinstance(mode, str) else mode
        Pp = _f64(P) if P is not None else None
        self.lib._check(self.lib._ivf_query_batch(
            self.h, _nullable(Pp), int(P is not None), _nullable(Qt), _nullable(Qr), nq, K, nprobe,
            m, eps0, delta_d, nthreads, ids, dists, dims, C.byref(secs)))
        return ids, dists, dims, secs.value

    def save(self, path):
        self.lib._check(self.lib._save_ivf(self.h, str(path).encode()))


class RefLib(_Common):
    """The reference library compiled from /root/reference (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self._fn("ref_ivf_build", [_f32p, _f32p, C.c_int32, C.c_int32, _f64p, C.c_int32,
                                   C.c_uint64, C.c_int, C.c_int32], _vp)
        self._fn("ref_ivf_assemble", [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int,
                                      C.c_uint64, _f64p, _f32p, _i32p, _f32p, _f32p], _vp)
        self._fn("ref_ivf_assemble_split", [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                            _f32p, _i32p, _f32p], _vp)
        self._fn("ref_ivf_from_split_layout", [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                               _f32p, _i64p, _i32p, _f32p, _f32p], _vp)
        self._fn("ref_ivf_free", [_vp], None)
        L = self.lib
        L.ref_hnsw_build.argtypes = [_f32p, _f32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64]
        L.ref_hnsw_build.restype = _vp
        L.ref_hnsw_load.argtypes = [C.c_char_p, _f32p, _f32p, C.c_int32, C.c_int32]
        L.ref_hnsw_load.restype = _vp
        L.ref_hnsw_save.argtypes = [_vp, C.c_char_p]
        L.ref_hnsw_free.argtypes = [_vp]
        L.ref_hnsw_free.restype = None
        L.ref_hnsw_query.argtypes = [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double, C.c_int32, _i32p,
                                     _f64p, C.POINTER(C.c_int32), _u64p]
        self._fn("ref_ivf_meta", [_vp, _i64p])
        self._fn("ref_ivf_export", [_vp] + [_vp] * 10)
        self._fn("ref_save_ivf", [_vp, C.c_char_p])
        self._fn("ref_load_ivf", [C.c_char_p], _vp)
        self._fn("ref_ivf_query", [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int, C.c_double,
                                   C.c_int32, _i32p, _f64p, C.POINTER(C.c_int32), _u64p])
        self._fn("ref_ivf_query_batch", [_vp, _vp, C.c_int, _vp, _vp, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int, C.c_double, C.c_int32, C.c_int,
                                         _i32p, _f64p, _u64p, C.POINTER(C.c_double)])
        self._fn("ref_synth_dataset", [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_uint64,
                                       _f32p, _vp])
        self._fn("ref_verify_theory", [_f32p, C.c_int32, C.c_int32, _f32p, C.c_int32, C.c_int32,
                                       _f64p, C.c_int32, _f64p, _f64p, _u64p, _u64p])

    def _handle(self, h):
        if not h:
            msg = self._last_error().decode(errors="replace")
            raise ValueError(msg)
        return RefIndex(self, h)

    def build_ivf(self, raw, t, P, k, seed, split=False, d1=32):
        raw = _f32(raw)
        return self._handle(self._ivf_build(raw, _f32(t), raw.shape[0], raw.shape[1], _f64(P), k,
                                            seed, int(split), d1))

    def assemble_ivf(self, raw, t, P, centroids_t, assignment, seed=0, split=True, d1=32):
        raw = _f32(raw)
        n, d = raw.shape
        cent = _f32(centroids_t)
        return self._handle(self._ivf_assemble(n, d, cent.shape[0], d1, int(split), seed, _f64(P),
                                               cent, np.ascontiguousarray(assignment, np.int32),
                                               raw, _f32(t)))

    def hnsw_build(self, raw, t, M, ef, seed):
        raw, t = _f32(raw), _f32(t)
        h = self.lib.ref_hnsw_build(raw, t, raw.shape[0], raw.shape[1], M, ef, seed)
        if not h:
            self._check(2)
        return h

    def hnsw_load(self, path, raw, t):
        raw, t = _f32(raw), _f32(t)
        h = self.lib.ref_hnsw_load(str(path).encode(), raw, t, raw.shape[0], raw.shape[1])
        if not h:
            self._check(2)
        return h

    def hnsw_save(self, h, path):
        self._check(self.lib.ref_hnsw_save(h, str(path).encode()))

    def hnsw_free(self, h):
        self.lib.ref_hnsw_free(h)

    def hnsw_query(self, h, q_t, q_raw, K, nef, mode, eps0=2.1, delta_d=32):
        """mode 0 plain, 1 pd, 2 plus, 3 plusplus -> (ids, dists, [dims, dco, hops, cand])."""
        ids = np.empty(K, np.int32)
        dists = np.empty(K, np.float64)
        cnt = C.c_int32()
        st = np.zeros(4, np.uint64)
        self._check(self.lib.ref_hnsw_query(h, _nullable(None if q_t is None else _f32(q_t)),
                                            _nullable(None if q_raw is None else _f32(q_raw)), K, nef, mode,
                                            eps0, delta_d, ids, dists, C.byref(cnt), st))
        return ids[:cnt.value].copy(), dists[:cnt.value].copy(), st

    def assemble_split(self, t, centroids_t, assignment, seed=0, d1=32):
        """kAdSplit-only reference IvfIndex (centroids_t, buckets, ids_flat, a1_t, a2_t)
        from transformed rows by id and their list assignment."""
        t = _f32(t)
        n, d = t.shape
        k = centroids_t.shape[0]
        return self._handle(self._ivf_assemble_split(n, d, k, d1, seed, _f32(centroids_t),
                                                     np.ascontiguousarray(assignment, np.int32), t))

    def from_split_layout(self, centroids_t, list_off, ids_flat, a1_t, a2_t, seed=0):
        """kAdSplit-only reference IvfIndex from a bucket-major split layout."""
        a1_t, a2_t = _f32(a1_t), _f32(a2_t)
        n, d1 = a1_t.shape
        d = d1 + a2_t.shape[1]
        k = centroids_t.shape[0]
        return self._handle(self._ivf_from_split_layout(
            n, d, k, d1, seed, _f32(centroids_t), np.ascontiguousarray(list_off, np.int64),
            np.ascontiguousarray(ids_flat, np.int32), a1_t, a2_t))

    def load_ivf(self, path):
        return self._handle(self._load_ivf(str(path).encode()))

    def synth_dataset(self, n, d, blobs, spread, seed, with_centers=False):
        out = np.empty((n, d), np.float32)
        cent = np.empty((blobs, d), np.float32) if with_centers else None
        self._check(self._synth_dataset(n, d, blobs, spread, seed, out, _nullable(cent)))
        return (out, cent) if with_centers else out

    def verify_theory(self, X, Q, K, grid):
        X = _f32(X)
        Q = _f32(Q)
        grid = _f64(sorted(grid))
        G = len(grid)
        fr, ad = np.empty(G), np.empty(G)
        fails, pos = np.empty(G, np.uint64), np.empty(G, np.uint64)
        self._check(self._verify_theory(X, X.shape[0], X.shape[1], Q, Q.shape[0], K, grid, G,
                                        fr, ad, fails, pos))
        return grid, fr, ad, fails, pos


def _maybe_build():
    if not os.path.exists(ORACLE_SO) or (
        os.path.exists(os.path.join(HERE, "adsann_oracle.c"))
        and os.path.getmtime(os.path.join(HERE, "adsann_oracle.c")) > os.path.getmtime(ORACLE_SO)
    ):
        subprocess.run(["make", "-C", HERE, "restate"], check=True, capture_output=True)


_ORC = None
_REF = None


def load_oracle() -> Oracle:
    global _ORC
    if _ORC is None:
        _maybe_build()
        _ORC = Oracle()
    return _ORC


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref() -> RefLib:
    global _REF
    if _REF is None:
        _REF = RefLib()
    return _REF
