"""ctypes binding of the libhookcc_cuda.so C-ABI (include/hookcc_c.h).

This is plumbing: every call goes straight to the CUDA library.  There is no
CPU fallback anywhere in this package; loading fails loudly when the shared
library is missing and compute calls fail with HCC_ENODEV without a B200.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libhookcc_cuda.so"

HCC_OK, HCC_EINVAL, HCC_ENOMEM, HCC_ECUDA, HCC_ENCCL, HCC_ENOTSTAR, HCC_ENODEV, HCC_ERANGE = range(8)
ALGO_BASELINE, ALGO_BASELINE_MJ, ALGO_ATOMIC, ALGO_ADAPTIVE = range(4)
ALGOS = {"baseline": ALGO_BASELINE, "baseline-mj": ALGO_BASELINE_MJ,
         "atomic": ALGO_ATOMIC, "adaptive": ALGO_ADAPTIVE}
FLAG_FULL_PASSES, FLAG_HOST_LOOP, FLAG_NO_GRAPH, FLAG_CHECK_STAR = 0x1, 0x2, 0x4, 0x8
FLAG_HOOK_EVENTS = 0x10
ABI_VERSION = 4  # HCC_ABI_VERSION of include/hookcc_c.h
HOOK_KERNELS = {1: "k_hook_small", 2: "k_hook", 3: "k_hook_sum", 4: "k_hook_cas",
                5: "k_hook_legacy", 6: "k_hook_sumd"}
PHASE_HOOK, PHASE_COMPRESS = 0, 1

u64, u32, i32 = C.c_uint64, C.c_uint32, C.c_int
vp = C.c_void_p

PHASE_CB = C.CFUNCTYPE(None, vp, i32, vp)


class Opts(C.Structure):
    _fields_ = [("algo", i32), ("segments", u64), ("first_pass_segments", u64),
                ("max_threads", u64), ("flags", u32), ("observer", PHASE_CB),
                ("observer_user", vp)]


class Counters(C.Structure):
    _fields_ = [("hook_traversal_steps", u64), ("cas_failures", u64), ("jump_steps", u64)]


class Metrics(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("hook_ms", C.c_double), ("compress_ms", C.c_double),
                ("s", u64), ("segments_clamped", i32), ("outer_iterations", u64),
                ("counters", Counters), ("components", u64), ("n", u64), ("m", u64),
                ("passes", u64), ("edges_processed", u64), ("records", u64),
                ("used_device_loop", i32), ("kernels", u64), ("star0_bitmap", i32),
                ("wl_capacity", u64), ("wl_reruns", u32), ("reserved_m", u32)]


class SegmentRec(C.Structure):
    _fields_ = [("hook_ms", C.c_double), ("compress_ms", C.c_double), ("counters", Counters),
                ("edges_in", u64), ("edges_out", u64), ("hook_event_ms", C.c_double),
                ("hook_start_ms", C.c_double), ("hook_end_ms", C.c_double),
                ("compress_start_ms", C.c_double), ("compress_end_ms", C.c_double),
                ("hook_kernel", C.c_int32), ("reserved_", C.c_int32)]


class GraphStats(C.Structure):
    _fields_ = [("n", u64), ("m_stored", u64), ("m_unique", u64), ("avg_degree", C.c_double),
                ("max_degree", u64)]


class ShardMetrics(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("local_ms", C.c_double), ("merge_ms", C.c_double),
                ("span_ms", C.c_double), ("pairs_exported", u64), ("records_merged", u64),
                ("rehook_passes", u64), ("bitmap_bytes", u64), ("roots_linked", u64),
                ("device", i32),
                ("peer_access", i32)]


class HccError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hcc error {code}: {msg}")
        self.code = code


_lib = None

# name -> (restype, argtypes)
_SIGS = {
    "hcc_abi_version": (i32, []),
    "hcc_last_error": (C.c_char_p, []),
    "hcc_device_count": (i32, []),
    "hcc_create": (i32, [i32, C.POINTER(vp)]),
    "hcc_destroy": (i32, [vp]),
    "hcc_ctx_segments": (i32, [vp, vp, u64, C.POINTER(u64)]),
    "hcc_ctx_sm_count": (i32, [vp, C.POINTER(i32)]),
    "hcc_graph_from_edges_u64": (i32, [vp, vp, u64, u64, C.POINTER(vp)]),
    "hcc_graph_from_edges_u32": (i32, [vp, vp, u64, u64, C.POINTER(vp)]),
    "hcc_graph_from_csr": (i32, [vp, vp, vp, u64, C.POINTER(vp)]),
    "hcc_graph_assign_edges_u32": (i32, [vp, vp, vp, u64, u64]),
    "hcc_graph_upload_async": (i32, [vp, vp, vp, u64, u64]),
    "hcc_graph_generate": (i32, [vp, C.c_char_p, u64, C.POINTER(vp)]),
    "hcc_graph_info": (i32, [vp, C.POINTER(u64), C.POINTER(u64)]),
    "hcc_graph_download_u32": (i32, [vp, vp, vp, u64, u64]),
    "hcc_graph_checksum": (i32, [vp, vp, C.POINTER(u64)]),
    "hcc_graph_compute_stats": (i32, [vp, vp, C.POINTER(GraphStats)]),
    "hcc_graph_free": (i32, [vp]),
    "hcc_cc": (i32, [vp, vp, C.POINTER(Opts), vp, vp, C.POINTER(Metrics)]),
    "hcc_cc_u64": (i32, [vp, vp, C.POINTER(Opts), vp, vp, C.POINTER(Metrics)]),
    "hcc_choose_segment_count": (u64, [C.POINTER(GraphStats)]),
    "hcc_forest_create": (i32, [vp, u64, C.POINTER(vp)]),
    "hcc_forest_free": (i32, [vp]),
    "hcc_forest_size": (i32, [vp, C.POINTER(u64)]),
    "hcc_forest_reset": (i32, [vp]),
    "hcc_forest_download_u64": (i32, [vp, vp]),
    "hcc_forest_download_u32": (i32, [vp, vp]),
    "hcc_forest_upload_u64": (i32, [vp, vp]),
    "hcc_forest_load": (i32, [vp, u64, C.POINTER(u64)]),
    "hcc_forest_store": (i32, [vp, u64, u64]),
    "hcc_forest_cas": (i32, [vp, u64, C.POINTER(u64), u64, C.POINTER(i32)]),
    "hcc_forest_hook": (i32, [vp, u64, u64, C.POINTER(i32)]),
    "hcc_forest_jump": (i32, [vp, u64, C.POINTER(i32)]),
    "hcc_forest_atomic_hook": (i32, [vp, u64, u64, C.POINTER(Counters)]),
    "hcc_forest_multi_jump": (i32, [vp, u64, C.POINTER(Counters)]),
    "hcc_forest_multi_jump_range": (i32, [vp, u64, u64, i32, C.POINTER(Counters)]),
    "hcc_forest_is_star": (i32, [vp, C.POINTER(i32)]),
    "hcc_forest_check_bound": (i32, [vp, C.POINTER(i32)]),
    "hcc_forest_export": (i32, [vp, vp, vp, vp, u64, C.POINTER(u64)]),
    "hcc_forest_verify": (i32, [vp, vp, vp, C.POINTER(u64), C.POINTER(u64)]),
    "hcc_labels_compare": (i32, [vp, vp, vp, u64, C.POINTER(i32), C.POINTER(i32)]),
    "hcc_rehook": (i32, [vp, vp, vp, vp, u64, C.POINTER(Metrics)]),
    "hcc_rehook_rows": (i32, [vp, vp, vp, u64, u64, u64, vp, u64, C.POINTER(Metrics)]),
    "hcc_graph_generate_range": (i32, [vp, C.c_char_p, u64, u64, u64, C.POINTER(vp)]),
    "hcc_create_multi": (i32, [C.POINTER(i32), i32, C.POINTER(vp)]),
    "hcc_ctx_shards": (i32, [vp, C.POINTER(i32)]),
    "hcc_ctx_shard_metrics": (i32, [vp, vp, u64, C.POINTER(u64)]),
    "hcc_peer_open": (i32, [vp, u64, u64, i32, i32, vp]),
    "hcc_peer_connect": (i32, [vp, vp]),
    "hcc_peer_export": (i32, [vp, vp]),
    "hcc_peer_merge": (i32, [vp, vp, C.POINTER(Metrics), C.POINTER(i32)]),
    "hcc_peer_disconnect": (i32, [vp]),
    "hcc_peer_close": (i32, [vp]),
}

PEER_HANDLE_BYTES = 256


def exported_symbols() -> list[str]:
    return list(_SIGS)


def lib() -> C.CDLL:
    """Load libhookcc_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("HCC_LIB", LIB_PATH))
        if not path.exists():
            raise ImportError(f"{path} not built; run `python -m paper_1612_01178_b200.build`")
        L = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.hcc_abi_version() != ABI_VERSION:  # structs are mirrored below
            raise ImportError(f"{path}: ABI {L.hcc_abi_version()} != binding ABI {ABI_VERSION}")
        _lib = L
    return _lib


def check(code: int) -> None:
    if code != HCC_OK:
        raise HccError(code, lib().hcc_last_error().decode())


def device_count() -> int:
    return lib().hcc_device_count()


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Context:
    """hcc_ctx: one device, stream and scratch (per host thread)."""

    def __init__(self, device: int = 0, devices: list[int] | None = None):
        """devices=[d0, d1, ...]: a multi-device context (hcc_create_multi),
        one edge shard per entry (entries may repeat)."""
        h = vp()
        if devices:
            arr = (i32 * len(devices))(*devices)
            check(lib().hcc_create_multi(arr, len(devices), C.byref(h)))
            device = devices[0]
        else:
            check(lib().hcc_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.devices = list(devices) if devices else [device]

    @property
    def shards(self) -> int:
        out = i32()
        check(lib().hcc_ctx_shards(self.h, C.byref(out)))
        return out.value

    def shard_metrics(self) -> list[dict]:
        cnt = u64()
        check(lib().hcc_ctx_shard_metrics(self.h, None, 0, C.byref(cnt)))
        arr = (ShardMetrics * max(cnt.value, 1))()
        check(lib().hcc_ctx_shard_metrics(self.h, C.cast(arr, vp), cnt.value, C.byref(cnt)))
        return [{k: getattr(arr[i], k) for k, _ in ShardMetrics._fields_}
                for i in range(cnt.value)]

    def close(self) -> None:
        if self.h:
            lib().hcc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def sm_count(self) -> int:
        out = i32()
        check(lib().hcc_ctx_sm_count(self.h, C.byref(out)))
        return out.value

    def segments(self) -> list[dict]:
        cnt = u64()
        check(lib().hcc_ctx_segments(self.h, None, 0, C.byref(cnt)))
        arr = (SegmentRec * max(cnt.value, 1))()
        check(lib().hcc_ctx_segments(self.h, C.cast(arr, vp), cnt.value, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            r = arr[i]
            out.append(dict(hook_ms=r.hook_ms, compress_ms=r.compress_ms,
                            hook_traversal_steps=r.counters.hook_traversal_steps,
                            cas_failures=r.counters.cas_failures,
                            jump_steps=r.counters.jump_steps,
                            edges_in=r.edges_in, edges_out=r.edges_out,
                            hook_event_ms=r.hook_event_ms,
                            hook_start_ms=r.hook_start_ms, hook_end_ms=r.hook_end_ms,
                            compress_start_ms=r.compress_start_ms,
                            compress_end_ms=r.compress_end_ms,
                            hook_kernel=HOOK_KERNELS.get(r.hook_kernel, "unknown")))
        return out

    # -- graphs --
    def graph_from_edges(self, edges: np.ndarray, n: int) -> "Graph":
        """edges: (m, 2) array of uint32 or uint64 endpoint pairs."""
        e = np.ascontiguousarray(edges)
        if e.ndim != 2 or (e.size and e.shape[1] != 2):
            raise ValueError("edges must have shape (m, 2)")
        m = e.shape[0]
        h = vp()
        if e.dtype == np.uint32:
            check(lib().hcc_graph_from_edges_u32(self.h, _ptr(e) if m else None, m, n, C.byref(h)))
        else:
            e = np.ascontiguousarray(e, dtype=np.uint64)
            check(lib().hcc_graph_from_edges_u64(self.h, _ptr(e) if m else None, m, n, C.byref(h)))
        return Graph(self, h)

    def graph_from_csr(self, row_ptr: np.ndarray, col: np.ndarray) -> "Graph":
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        cl = np.ascontiguousarray(col, dtype=np.uint32)
        h = vp()
        check(lib().hcc_graph_from_csr(self.h, _ptr(rp), _ptr(cl) if cl.size else None,
                                       len(rp) - 1, C.byref(h)))
        return Graph(self, h)

    def generate(self, spec: str, default_seed: int = 1) -> "Graph":
        h = vp()
        check(lib().hcc_graph_generate(self.h, spec.encode(), default_seed, C.byref(h)))
        return Graph(self, h)

    def generate_range(self, spec: str, first: int, count: int, default_seed: int = 1) -> "Graph":
        """Edges [first, first+count) of a device generator spec (one shard)."""
        h = vp()
        check(lib().hcc_graph_generate_range(self.h, spec.encode(), default_seed, first, count,
                                             C.byref(h)))
        return Graph(self, h)

    # -- multi-process merge over CUDA IPC (hcc_peer_*) --
    def peer_open(self, n: int, cap: int, rank: int, world: int) -> bytes:
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        check(lib().hcc_peer_open(self.h, n, cap, rank, world, buf))
        return buf.raw

    def peer_connect(self, handles: bytes) -> None:
        buf = C.create_string_buffer(handles, len(handles))
        check(lib().hcc_peer_connect(self.h, buf))

    def peer_export(self, forest: "Forest") -> None:
        check(lib().hcc_peer_export(self.h, forest.h))

    def peer_merge(self, forest: "Forest") -> tuple[dict, bool]:
        mx = Metrics()
        ovf = i32()
        check(lib().hcc_peer_merge(self.h, forest.h, C.byref(mx), C.byref(ovf)))
        return metrics_dict(mx), bool(ovf.value)

    def peer_disconnect(self) -> None:
        check(lib().hcc_peer_disconnect(self.h))

    def peer_close(self) -> None:
        check(lib().hcc_peer_close(self.h))

    def export(self, forest: "Forest", dev_bits: int, dev_pairs: int, cap: int) -> int:
        """hcc_forest_export into caller device buffers; returns the pair count
        (may exceed cap: then retry with a larger buffer)."""
        cnt = u64()
        check(lib().hcc_forest_export(self.h, forest.h, dev_bits, dev_pairs, cap, C.byref(cnt)))
        return cnt.value

    def rehook(self, forest: "Forest", dev_bits_or: int | None, dev_pairs: int | None,
               count: int) -> dict:
        mx = Metrics()
        check(lib().hcc_rehook(self.h, forest.h, dev_bits_or, dev_pairs, count, C.byref(mx)))
        return metrics_dict(mx)

    def rehook_rows(self, forest: "Forest", dev_rows: int | None, nrows: int, stride: int,
                    skip: int, dev_pairs: int | None, count: int) -> dict:
        """hcc_rehook_rows: OR of the gathered bitmap rows but `skip` (-1: none)."""
        mx = Metrics()
        check(lib().hcc_rehook_rows(self.h, forest.h, dev_rows, nrows, stride,
                                    skip if skip >= 0 else 2**64 - 1, dev_pairs, count,
                                    C.byref(mx)))
        return metrics_dict(mx)

    def verify(self, graph: "Graph", forest: "Forest") -> tuple[int, int]:
        """(edges split by the labels, non-canonical vertices); (0, 0) when correct."""
        be, bv = u64(), u64()
        check(lib().hcc_forest_verify(self.h, graph.h, forest.h, C.byref(be), C.byref(bv)))
        return be.value, bv.value

    def labels_compare(self, a: np.ndarray, b: np.ndarray) -> tuple[bool, bool]:
        """(partitions equal, arrays equal) computed on the device."""
        x = np.ascontiguousarray(a, dtype=np.uint32)
        y = np.ascontiguousarray(b, dtype=np.uint32)
        if x.shape != y.shape:
            raise ValueError("partitions_equal: length mismatch")
        pe, ex = i32(), i32()
        check(lib().hcc_labels_compare(self.h, _ptr(x) if x.size else None,
                                       _ptr(y) if y.size else None, x.size,
                                       C.byref(pe), C.byref(ex)))
        return bool(pe.value), bool(ex.value)

    def forest(self, n: int) -> "Forest":
        h = vp()
        check(lib().hcc_forest_create(self.h, n, C.byref(h)))
        return Forest(self, h, n)

    # -- the CC entry point --
    def cc(self, graph: "Graph", algo: str | int = "baseline-mj", segments: int = 0,
           first_pass_segments: int = 0, max_threads: int = 0, flags: int = 0,
           forest: "Forest | None" = None, labels: bool = True, observer=None,
           labels_out: np.ndarray | None = None):
        """Run connected components; returns (labels u32 | None, metrics dict)."""
        a = ALGOS[algo] if isinstance(algo, str) else int(algo)
        cb = PHASE_CB(0)
        if observer is not None:
            def _cb(user, phase, fh, _obs=observer, _n=graph.n):
                _obs(phase, Forest(self, vp(fh), _n, owned=False))
            cb = PHASE_CB(_cb)
        o = Opts(a, segments, first_pass_segments, max_threads, flags, cb, None)
        mx = Metrics()
        out = None
        if labels:
            out = labels_out if labels_out is not None else np.empty(graph.n, dtype=np.uint32)
        check(lib().hcc_cc(self.h, graph.h, C.byref(o), forest.h if forest else None,
                           _ptr(out) if (out is not None and graph.n) else None, C.byref(mx)))
        return out, metrics_dict(mx)


def metrics_dict(mx: Metrics) -> dict:
    return dict(total_ms=mx.total_ms, hook_ms=mx.hook_ms, compress_ms=mx.compress_ms,
                s=mx.s, segments_clamped=bool(mx.segments_clamped),
                outer_iterations=mx.outer_iterations,
                hook_traversal_steps=mx.counters.hook_traversal_steps,
                cas_failures=mx.counters.cas_failures, jump_steps=mx.counters.jump_steps,
                components=mx.components, n=mx.n, m=mx.m, passes=mx.passes,
                edges_processed=mx.edges_processed, records=mx.records,
                used_device_loop=bool(mx.used_device_loop), kernels=mx.kernels,
                star0_bitmap=bool(mx.star0_bitmap), wl_capacity=mx.wl_capacity,
                wl_reruns=mx.wl_reruns)


class Graph:
    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h
        n, m = u64(), u64()
        check(lib().hcc_graph_info(h, C.byref(n), C.byref(m)))
        self.n, self.m = n.value, m.value

    def close(self):
        if self.h:
            lib().hcc_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def edges(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.m - first if count is None else count
        out = np.empty((count, 2), dtype=np.uint32)
        check(lib().hcc_graph_download_u32(self.ctx.h, self.h, _ptr(out) if count else None,
                                           first, count))
        return out

    def assign(self, edges: np.ndarray, first: int = 0) -> None:
        """Overwrite edges [first, first+len) from host u32 pairs (pinned memory
        gives full PCIe bandwidth)."""
        e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        check(lib().hcc_graph_assign_edges_u32(self.ctx.h, self.h, _ptr(e) if e.size else None,
                                               first, e.shape[0]))

    def upload_async(self, edges: np.ndarray, first: int = 0) -> None:
        """hcc_graph_upload_async: refill edges [first, first+len) on the copy
        stream and return at once (`edges` must stay alive and unchanged until
        the next call that reads this graph; pinned memory for overlap)."""
        e = edges.reshape(-1, 2)
        if e.dtype != np.uint32 or not e.flags["C_CONTIGUOUS"]:
            raise ValueError("upload_async needs a C-contiguous uint32 (m, 2) array")
        check(lib().hcc_graph_upload_async(self.ctx.h, self.h, _ptr(e) if e.size else None,
                                           first, e.shape[0]))

    def checksum(self) -> int:
        out = u64()
        check(lib().hcc_graph_checksum(self.ctx.h, self.h, C.byref(out)))
        return out.value

    def stats(self) -> dict:
        st = GraphStats()
        check(lib().hcc_graph_compute_stats(self.ctx.h, self.h, C.byref(st)))
        return dict(n=st.n, m_stored=st.m_stored, m_unique=st.m_unique,
                    avg_degree=st.avg_degree, max_degree=st.max_degree)


class Forest:
    """Device ParentForest (forest.hpp:19-63)."""

    def __init__(self, ctx: Context, h, n: int, owned: bool = True):
        self.ctx, self.h, self.n, self.owned = ctx, h, n, owned

    def close(self):
        if self.h and self.owned:
            lib().hcc_forest_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        check(lib().hcc_forest_reset(self.h))

    def snapshot(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint64)
        check(lib().hcc_forest_download_u64(self.h, _ptr(out) if self.n else None))
        return out

    def snapshot_u32(self) -> np.ndarray:
        return self.download_u32(np.empty(self.n, dtype=np.uint32))

    def download_u32(self, out: np.ndarray) -> np.ndarray:
        """The labels as u32 into a caller buffer (pinned for full PCIe speed)."""
        assert out.dtype == np.uint32 and out.size >= self.n and out.flags["C_CONTIGUOUS"]
        check(lib().hcc_forest_download_u32(self.h, _ptr(out) if self.n else None))
        return out

    def upload(self, parents) -> None:
        a = np.ascontiguousarray(parents, dtype=np.uint64)
        check(lib().hcc_forest_upload_u64(self.h, _ptr(a) if self.n else None))

    def load(self, v: int) -> int:
        out = u64()
        check(lib().hcc_forest_load(self.h, v, C.byref(out)))
        return out.value

    def store(self, v: int, p: int) -> None:
        check(lib().hcc_forest_store(self.h, v, p))

    def cas(self, v: int, expected: int, desired: int):
        e = u64(expected)
        ok = i32()
        check(lib().hcc_forest_cas(self.h, v, C.byref(e), desired, C.byref(ok)))
        return bool(ok.value), e.value

    def hook(self, u: int, v: int) -> bool:
        ch = i32()
        check(lib().hcc_forest_hook(self.h, u, v, C.byref(ch)))
        return bool(ch.value)

    def jump(self, v: int) -> bool:
        ch = i32()
        check(lib().hcc_forest_jump(self.h, v, C.byref(ch)))
        return bool(ch.value)

    def atomic_hook(self, u: int, v: int, counters: Counters) -> None:
        check(lib().hcc_forest_atomic_hook(self.h, u, v, C.byref(counters)))

    def multi_jump(self, v: int, counters: Counters) -> None:
        check(lib().hcc_forest_multi_jump(self.h, v, C.byref(counters)))

    def multi_jump_range(self, begin: int, end: int, descending: bool, counters: Counters) -> None:
        check(lib().hcc_forest_multi_jump_range(self.h, begin, end, int(descending), C.byref(counters)))

    def is_star(self) -> bool:
        out = i32()
        check(lib().hcc_forest_is_star(self.h, C.byref(out)))
        return bool(out.value)

    def bound_ok(self) -> bool:
        out = i32()
        check(lib().hcc_forest_check_bound(self.h, C.byref(out)))
        return bool(out.value)
