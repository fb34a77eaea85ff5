"""CPU parity checkers for the B200 hookcc library — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
`--impl reference` arm) may import this package, and only as the checker or
the reported CPU baseline.  The product path (paper_1612_01178_b200 and
libhookcc_cuda.so) never imports or links it.

Two libraries:
  * liboracle.so — oracle/hookcc_oracle.c, a plain-C restatement of the
    reference algorithm (each function cites the reference file:line).
  * _ref/libhookcc_ref.so — the unmodified reference headers compiled from
    /root/reference by oracle/Makefile (ref_harness.cpp wraps their API).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libhookcc_ref.so"

u64, u32, i32, dbl, vp = C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_void_p


class RunOut(C.Structure):
    _fields_ = [("outer_iterations", u64), ("s", u64), ("clamped", i32),
                ("hook_traversal_steps", u64), ("cas_failures", u64), ("jump_steps", u64),
                ("components", u64)]


class RefMetrics(C.Structure):
    _fields_ = [("total_ms", dbl), ("hook_ms", dbl), ("compress_ms", dbl), ("s", u64),
                ("outer_iterations", u64), ("hook_traversal_steps", u64),
                ("cas_failures", u64), ("jump_steps", u64), ("components", u64),
                ("segments_clamped", i32), ("workers", C.c_uint)]


_O = None
_R = None


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _olib() -> C.CDLL:
    global _O
    if _O is None:
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO))
        sig = {
            "oracle_gen_er": (i32, [u64, u64, u64, vp]),
            "oracle_gen_rmat": (i32, [u32, u64, dbl, dbl, dbl, dbl, u64, vp]),
            "oracle_gen_grid": (i32, [u64, u64, vp]),
            "oracle_gen_rmatx": (None, [u32, dbl, dbl, dbl, u64, u64, u64, vp]),
            "oracle_gen_erx": (None, [u64, u64, u64, u64, vp]),
            "oracle_checksum_u32": (u64, [vp, u64, u64]),
            "oracle_cc_u64": (i32, [u64, vp, u64, vp]),
            "oracle_cc_u32": (i32, [u64, vp, u64, vp]),
            "oracle_cc_stream": (i32, [i32, u32, dbl, dbl, dbl, u64, u64, u64, u64, i32, vp,
                                       C.POINTER(u64), C.POINTER(u64)]),
            "oracle_bfs_cc_u64": (i32, [u64, vp, u64, vp]),
            "oracle_hook": (i32, [vp, u64, u64]),
            "oracle_jump": (i32, [vp, u64]),
            "oracle_atomic_hook": (None, [vp, u64, u64, vp]),
            "oracle_multi_jump": (None, [vp, u64, vp]),
            "oracle_is_star": (i32, [vp, u64]),
            "oracle_baseline_cc": (i32, [u64, vp, u64, vp, C.POINTER(RunOut)]),
            "oracle_baseline_mj_cc": (i32, [u64, vp, u64, vp, C.POINTER(RunOut)]),
            "oracle_adaptive_cc": (i32, [u64, vp, u64, u64, vp, C.POINTER(RunOut), vp]),
            "oracle_partition": (u64, [u64, u64, vp, C.POINTER(i32)]),
            "oracle_stats_u64": (i32, [u64, vp, u64, C.POINTER(u64), C.POINTER(u64)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _O = L
    return _O


def ref_available() -> bool:
    return REF_SO.exists()


def _rlib() -> C.CDLL:
    global _R
    if _R is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; make -C oracle)")
        L = C.CDLL(str(REF_SO))
        sig = {
            "ref_hardware_workers": (C.c_uint, []),
            "ref_gen_er": (i32, [u64, u64, u64, vp]),
            "ref_gen_rmat": (i32, [C.c_uint, u64, dbl, dbl, dbl, dbl, u64, vp]),
            "ref_gen_grid": (i32, [u64, u64, vp]),
            "ref_oracle_cc": (i32, [u64, vp, u64, vp]),
            "ref_bfs_cc": (i32, [u64, vp, u64, vp]),
            "ref_stats": (i32, [u64, vp, u64, C.POINTER(u64), C.POINTER(dbl), C.POINTER(u64)]),
            "ref_choose_segment_count": (u64, [u64, u64, dbl]),
            "ref_run": (i32, [i32, u64, vp, u64, u64, C.c_uint, vp, C.POINTER(RefMetrics), vp, u64]),
            "ref_graph_new32": (vp, [u64, vp, u64]),
            "ref_graph_free": (None, [vp]),
            "ref_run_graph": (i32, [i32, vp, u64, C.c_uint, vp, C.POINTER(RefMetrics)]),
            "ref_hook": (i32, [vp, u64, u64, u64]),
            "ref_jump": (i32, [vp, u64, u64]),
            "ref_atomic_hook": (None, [vp, u64, u64, u64, vp]),
            "ref_multi_jump": (None, [vp, u64, u64, vp]),
            "ref_is_star": (i32, [vp, u64]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _R = L
    return _R


def _p(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _e64(edges) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint64).reshape(-1, 2))
    return e


# ---------------------------------------------------------------- restatement
def gen_er(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty((m, 2), dtype=np.uint64)
    if _olib().oracle_gen_er(n, m, seed, _p(out)):
        raise ValueError("erdos_renyi: zero vertices")
    return out


def gen_rmat(scale: int, ef: int, seed: int, a=0.57, b=0.19, c=0.19, d=0.05) -> np.ndarray:
    m = ef << scale
    out = np.empty((m, 2), dtype=np.uint64)
    if _olib().oracle_gen_rmat(scale, ef, a, b, c, d, seed, _p(out)):
        raise ValueError("rmat: quadrant probabilities must sum to 1")
    return out


def gen_grid(rows: int, cols: int) -> np.ndarray:
    m = rows * (cols - 1) + (rows - 1) * cols
    out = np.empty((m, 2), dtype=np.uint64)
    if _olib().oracle_gen_grid(rows, cols, _p(out)):
        raise ValueError("grid: zero vertices")
    return out


def gen_rmatx(scale: int, seed: int, first: int, count: int, a=0.57, b=0.19, c=0.19) -> np.ndarray:
    out = np.empty((count, 2), dtype=np.uint32)
    _olib().oracle_gen_rmatx(scale, a, b, c, seed, first, count, _p(out))
    return out


def gen_erx(n: int, seed: int, first: int, count: int) -> np.ndarray:
    out = np.empty((count, 2), dtype=np.uint32)
    _olib().oracle_gen_erx(n, seed, first, count, _p(out))
    return out


def checksum_u32(uv: np.ndarray, first: int = 0) -> int:
    e = np.ascontiguousarray(uv, dtype=np.uint32)
    return _olib().oracle_checksum_u32(_p(e), first, e.shape[0])


def cc(n: int, edges) -> np.ndarray:
    """oracle_cc (oracle.hpp:47-62) -> min-canonical labels."""
    e = np.asarray(edges)
    if e.dtype == np.uint32:
        e = np.ascontiguousarray(e.reshape(-1, 2))
        out = np.empty(n, dtype=np.uint32)
        if _olib().oracle_cc_u32(n, _p(e), e.shape[0], _p(out)):
            raise ValueError("endpoint out of range")
        return out
    e = _e64(e)
    out = np.empty(n, dtype=np.uint64)
    if _olib().oracle_cc_u64(n, _p(e), e.shape[0], _p(out)):
        raise ValueError("endpoint out of range")
    return out


def cc_stream(spec: str, first: int = 0, count: int | None = None, threads: int = 0):
    """Streaming oracle_cc over a counter-based generator spec (rmatx / erx),
    never materialising the edges: -> (labels u32, edge checksum, components).
    For graphs too large to hold (RMAT-28: 2^32 edges, 1 GiB of labels)."""
    import os
    kind, params = spec.split(":", 1)
    kv = dict(p.split("=") for p in params.split(","))
    seed = int(kv.get("seed", 1))
    if kind == "rmatx":
        scale, ef = int(kv["scale"]), int(kv["ef"])
        n, m, k, n_er = 1 << scale, ef << scale, 0, 0
        a, b, c = float(kv.get("a", 0.57)), float(kv.get("b", 0.19)), float(kv.get("c", 0.19))
    elif kind == "erx":
        n, m, k, scale = int(kv["n"]), int(kv["m"]), 1, 0
        n_er, a, b, c = n, 0.0, 0.0, 0.0
    else:
        raise ValueError(f"cc_stream: unsupported generator `{kind}`")
    count = m - first if count is None else count
    out = np.empty(n, dtype=np.uint32)
    ck, comp = u64(), u64()
    rc = _olib().oracle_cc_stream(k, scale, a, b, c, n_er, seed, first, count,
                                  threads or (os.cpu_count() or 1), _p(out), C.byref(ck),
                                  C.byref(comp))
    if rc:
        raise RuntimeError(f"oracle_cc_stream failed ({rc})")
    return out, ck.value, comp.value


def bfs_cc(n: int, edges) -> np.ndarray:
    e = _e64(edges)
    out = np.empty(n, dtype=np.uint64)
    _olib().oracle_bfs_cc_u64(n, _p(e), e.shape[0], _p(out))
    return out


def stats(n: int, edges) -> dict:
    e = _e64(edges)
    uq, mx = u64(), u64()
    _olib().oracle_stats_u64(n, _p(e), e.shape[0], C.byref(uq), C.byref(mx))
    return dict(n=n, m_stored=e.shape[0], m_unique=uq.value,
                avg_degree=(2.0 * uq.value / n) if n else 0.0, max_degree=mx.value)


def run_seq(algo: str, n: int, edges, segments: int = 1):
    """Sequential (workers = 1) drivers -> (labels, RunOut, seg_counters)."""
    e = _e64(edges)
    pi = np.empty(max(n, 1), dtype=np.uint64)
    r = RunOut()
    segc = None
    L = _olib()
    if algo == "baseline":
        L.oracle_baseline_cc(n, _p(e), e.shape[0], _p(pi), C.byref(r))
    elif algo == "baseline-mj":
        L.oracle_baseline_mj_cc(n, _p(e), e.shape[0], _p(pi), C.byref(r))
    else:
        s = 1 if algo == "atomic" else segments
        segc = np.zeros(3 * max(1, min(max(s, 1), max(e.shape[0], 1))), dtype=np.uint64)
        L.oracle_adaptive_cc(n, _p(e), e.shape[0], s, _p(pi), C.byref(r), _p(segc))
    return pi[:n].copy(), r, segc


# --------------------------------------------------------------- reference
def ref_workers() -> int:
    return _rlib().ref_hardware_workers()


def ref_gen_rmat(scale: int, ef: int, seed: int, a=0.57, b=0.19, c=0.19, d=0.05) -> np.ndarray:
    out = np.empty((ef << scale, 2), dtype=np.uint64)
    if _rlib().ref_gen_rmat(scale, ef, a, b, c, d, seed, _p(out)):
        raise ValueError("rmat failed")
    return out


def ref_gen_er(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty((m, 2), dtype=np.uint64)
    if _rlib().ref_gen_er(n, m, seed, _p(out)):
        raise ValueError("erdos_renyi failed")
    return out


def ref_gen_grid(rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows * (cols - 1) + (rows - 1) * cols, 2), dtype=np.uint64)
    if _rlib().ref_gen_grid(rows, cols, _p(out)):
        raise ValueError("grid failed")
    return out


def ref_cc(n: int, edges) -> np.ndarray:
    e = _e64(edges)
    out = np.empty(n, dtype=np.uint64)
    _rlib().ref_oracle_cc(n, _p(e), e.shape[0], _p(out))
    return out


def ref_bfs_cc(n: int, edges) -> np.ndarray:
    e = _e64(edges)
    out = np.empty(n, dtype=np.uint64)
    _rlib().ref_bfs_cc(n, _p(e), e.shape[0], _p(out))
    return out


def ref_stats(n: int, edges) -> dict:
    e = _e64(edges)
    uq, avg, mx = u64(), dbl(), u64()
    _rlib().ref_stats(n, _p(e), e.shape[0], C.byref(uq), C.byref(avg), C.byref(mx))
    return dict(n=n, m_stored=e.shape[0], m_unique=uq.value, avg_degree=avg.value,
                max_degree=mx.value)


REF_ALGOS = {"baseline": 0, "baseline-mj": 1, "atomic": 2, "adaptive": 3}


def ref_run(algo: str, n: int, edges, segments: int = 0, workers: int = 0, seg_cap: int = 0):
    """Run a reference engine -> (labels u64, metrics dict, seg_counters)."""
    e = _e64(edges)
    lab = np.empty(max(n, 1), dtype=np.uint64)
    mx = RefMetrics()
    segc = np.zeros(3 * max(seg_cap, 1), dtype=np.uint64)
    rc = _rlib().ref_run(REF_ALGOS[algo], n, _p(e), e.shape[0], segments, workers, _p(lab),
                         C.byref(mx), _p(segc) if seg_cap else None, seg_cap)
    if rc:
        raise RuntimeError(f"reference run failed ({rc})")
    return lab[:n].copy(), _ref_metrics(mx), segc[:3 * seg_cap].reshape(-1, 3) if seg_cap else None


def _ref_metrics(mx: RefMetrics) -> dict:
    return {k: getattr(mx, k) for k, _ in RefMetrics._fields_}


class RefGraph:
    """A reference hookcc::Graph built once from packed u32 edges."""

    def __init__(self, n: int, uv32: np.ndarray):
        e = np.ascontiguousarray(uv32, dtype=np.uint32)
        self.h = _rlib().ref_graph_new32(n, _p(e), e.shape[0])
        if not self.h:
            raise MemoryError("reference Graph allocation failed")
        self.n = n

    def run(self, algo: str, segments: int = 0, workers: int = 0, labels: bool = False):
        lab = np.empty(max(self.n, 1), dtype=np.uint64) if labels else None
        mx = RefMetrics()
        rc = _rlib().ref_run_graph(REF_ALGOS[algo], self.h, segments, workers,
                                   _p(lab) if labels else None, C.byref(mx))
        if rc:
            raise RuntimeError(f"reference run failed ({rc})")
        return (lab[:self.n] if labels else None), _ref_metrics(mx)

    def close(self):
        if self.h:
            _rlib().ref_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_elem(op: str, pi, *args):
    """Run a reference forest.hpp kernel on a host copy; returns (result, pi, counters)."""
    p = np.ascontiguousarray(np.asarray(pi, dtype=np.uint64)).copy()
    n = p.shape[0]
    cnt = np.zeros(3, dtype=np.uint64)
    L = _rlib()
    res = None
    if op == "hook":
        res = bool(L.ref_hook(_p(p), n, *args))
    elif op == "jump":
        res = bool(L.ref_jump(_p(p), n, *args))
    elif op == "atomic_hook":
        L.ref_atomic_hook(_p(p), n, args[0], args[1], _p(cnt))
    elif op == "multi_jump":
        L.ref_multi_jump(_p(p), n, args[0], _p(cnt))
    elif op == "is_star":
        res = bool(L.ref_is_star(_p(p), n))
    return res, p, cnt
