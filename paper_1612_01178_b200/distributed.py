"""Edge-partitioned multi-GPU connected components (north-star (5)).

One process per GPU.  Rank r owns the contiguous edge range
partition_edges(m, world)[r] (engines.hpp:43-58: the first m % world ranks
get one extra edge) and runs the single-GPU Hook-Compress engine on it into
a full local forest (stars).  The merge is one exchange round (§8e shape 3):

  1. export   each rank encodes its forest as a bitmap of {v : pi(v) == 0}
              (the giant component's root on skewed graphs) plus sparse
              (v, pi(v)) pairs for the remaining non-self entries;
  2. exchange the peers' payloads reach every rank;
  3. re-hook  each rank hooks the remote relations as (v, pi_remote(v)) edges
              into its own forest with the worklist engine.

Two transports for step 2:
  * PeerMerge (default on GPUs): CUDA IPC.  Every rank maps its peers'
    export arenas once (hcc_peer_open / hcc_peer_connect; the handle blobs
    are all-gathered over the process group), and per run the merge kernel
    (k_merge_gather) reads them in place over NVLink -- steps 2 and 3 are one
    kernel plus the re-hook passes; the host only runs one barrier between
    export and merge and a one-int all-reduce (pair-buffer overflow) after.
    The same kernel serves the single-process multi-device context
    (hcc_create_multi).
  * merge_round (NCCL / gloo): all-gather of the bitmaps (OR-combined) and of
    the pair lists (sizes first, then the padded payloads); the protocol is
    testable on CPU with gloo.

After the round every rank holds the union of all shards' relations, i.e. the
global min-canonical labels.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np


def edge_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """(first, count) of rank's shard under partition_edges(m, world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(m, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


@dataclass
class MergeTimes:
    local_ms: float = 0.0
    export_ms: float = 0.0
    exchange_ms: float = 0.0
    rehook_ms: float = 0.0
    pairs_sent: int = 0
    pairs_received: int = 0
    bits_bytes: int = 0
    rehook_passes: int = 0
    extra: dict = field(default_factory=dict)


_BUFS: dict = {}


def _buf(key, numel, dtype, device):
    """Reusable receive buffers, one per (key, dtype, device), grown
    geometrically: the exchange runs every step with varying pair counts."""
    import torch
    k = (key, dtype, str(device))
    t = _BUFS.get(k)
    if t is None or t.numel() < numel:
        t = torch.empty(max(numel, (t.numel() * 3 // 2) if t is not None else 0),
                        dtype=dtype, device=device)
        _BUFS[k] = t
    return t[:numel]


def send_offset(nwords: int) -> int:
    """Index of the pair count in the send buffer (8-byte aligned)."""
    return nwords + (nwords & 1)


def exchange(bits, pairs, group=None, sendbuf=None, pairs_buf=None):
    """All-gather the payloads: two collectives and one host read.

    bits      : int32 tensor [nwords] (bit patterns), this rank's bitmap
    pairs     : int32 tensor [k, 2], this rank's (v, parent) pairs
    sendbuf   : optional int32 [send_offset(nwords) + 2] whose prefix is
                `bits`: the pair count rides in its last two words (no extra
                collective)
    pairs_buf : optional [cap, 2] tensor whose prefix is `pairs`: sent as is
                (rows past k are ignored by the receivers), no padding copy
    returns (rows, rank, remote): the gathered bitmaps as [world, nwords]
    (the receiver ORs every row but its own), and the remote pairs [K, 2].
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = bits.device
    nw = bits.numel()
    off = send_offset(nw)
    k = int(pairs.shape[0])
    if sendbuf is None or sendbuf.numel() != off + 2:
        sendbuf = torch.zeros(off + 2, dtype=torch.int32, device=dev)
        sendbuf[:nw] = bits
    sendbuf[off:].view(torch.int64).fill_(k)
    gathered = _buf("bits", world * (off + 2), torch.int32, dev)
    dist.all_gather_into_tensor(gathered, sendbuf, group=group)
    gathered = gathered.view(world, off + 2)
    sizes_h = gathered[:, off:].contiguous().view(torch.int64).view(-1).cpu().tolist()
    rows = gathered[:, :nw]
    kmax = max(sizes_h) if sizes_h else 0
    if kmax == 0:
        return rows, rank, torch.empty((0, 2), dtype=pairs.dtype, device=dev)
    if pairs_buf is not None and pairs_buf.shape[0] >= kmax:
        send = pairs_buf[:kmax]
    else:
        send = torch.zeros((kmax, 2), dtype=pairs.dtype, device=dev)
        send[:k] = pairs
    allp = _buf("pairs", world * kmax * 2, pairs.dtype, dev)
    dist.all_gather_into_tensor(allp, send.contiguous().view(-1), group=group)
    allp = allp.view(world * kmax, 2)
    parts = [allp[r * kmax: r * kmax + sizes_h[r]] for r in range(world) if r != rank and sizes_h[r]]
    remote = torch.cat(parts) if parts else torch.empty((0, 2), dtype=pairs.dtype, device=dev)
    return rows, rank, remote


def or_rows(rows, rank):
    """OR of the gathered bitmap rows except `rank`'s (backends without a
    row-aware re-hook)."""
    import torch
    out = torch.zeros_like(rows[0])
    for r in range(rows.shape[0]):
        if r != rank:
            out.bitwise_or_(rows[r])
    return out


def merge_round(backend, group=None, sync=None) -> MergeTimes:
    """export -> exchange -> re-hook on this rank (local CC already done)."""
    t = MergeTimes()
    sync = sync or (lambda: None)
    t0 = time.perf_counter()
    bits, pairs = backend.export()
    sync()
    t1 = time.perf_counter()
    rows, rank, remote = exchange(bits, pairs, group, getattr(backend, "sendbuf", None),
                                  getattr(backend, "pairs", None))
    sync()
    t2 = time.perf_counter()
    if hasattr(backend, "rehook_rows"):
        mx = backend.rehook_rows(rows, rank, remote)
    else:
        mx = backend.rehook(or_rows(rows, rank), remote)
    sync()
    t3 = time.perf_counter()
    t.export_ms, t.exchange_ms, t.rehook_ms = 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)
    t.pairs_sent = int(pairs.shape[0])
    t.pairs_received = int(remote.shape[0])
    t.bits_bytes = int(bits.numel() * 4)
    t.rehook_passes = int(mx.get("passes", 0)) if isinstance(mx, dict) else 0
    return t


class CudaBackend:
    """The B200 path: libhookcc_cuda.so kernels on torch CUDA buffers."""

    def __init__(self, ctx, n: int, device):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.n = n
        self.device = device
        self.forest = ctx.forest(n)
        self.nwords = (n + 31) // 32
        # the exported bitmap is the prefix of the exchange's send buffer
        self.sendbuf = torch.zeros(send_offset(self.nwords) + 2, dtype=torch.int32,
                                   device=device)
        self.bits = self.sendbuf[: self.nwords]
        self.cap = max(1 << 16, n // 64)
        self.pairs = torch.empty((self.cap, 2), dtype=torch.int32, device=device)
        self.local_metrics = None

    def local_cc(self, graph, **kw):
        _, self.local_metrics = self.ctx.cc(graph, "baseline-mj", forest=self.forest,
                                            labels=False, **kw)
        return self.local_metrics

    def export(self):
        k = self.ctx.export(self.forest, self.bits.data_ptr(), self.pairs.data_ptr(), self.cap)
        if k > self.cap:
            self.cap = k + (k >> 3)
            self.pairs = self.torch.empty((self.cap, 2), dtype=self.torch.int32,
                                          device=self.device)
            k = self.ctx.export(self.forest, self.bits.data_ptr(), self.pairs.data_ptr(), self.cap)
        return self.bits, self.pairs[:k]

    def rehook(self, bits_or, remote):
        remote = remote.contiguous()
        # the gathered buffers were written on torch's stream; the library
        # reads them on its own stream
        self.torch.cuda.current_stream().synchronize()
        return self.ctx.rehook(self.forest, bits_or.data_ptr(),
                               remote.data_ptr() if remote.shape[0] else None,
                               int(remote.shape[0]))

    def rehook_rows(self, rows, rank, remote):
        # rows: [world, nwords] view of the gathered buffer (row stride
        # send_offset(nwords) + 2)
        remote = remote.contiguous()
        self.torch.cuda.current_stream().synchronize()
        return self.ctx.rehook_rows(self.forest, rows.data_ptr(), int(rows.shape[0]),
                                    int(rows.stride(0)), int(rank),
                                    remote.data_ptr() if remote.shape[0] else None,
                                    int(remote.shape[0]))

    def labels(self) -> np.ndarray:
        return self.forest.snapshot()


class PeerUnavailable(RuntimeError):
    """The CUDA-IPC transport cannot be set up on every rank (raised on all
    ranks together)."""


class PeerMerge:
    """Merge over CUDA IPC (hcc_peer_*): k_merge_gather reads the peers'
    export arenas in place over NVLink.  Host traffic per run: one barrier
    between export and merge (every export event is recorded before any
    rank waits on it) and a one-int MAX all-reduce after the merge, which
    also keeps a fast rank's next export from overwriting an arena a slow
    rank is still reading.  A rank whose pair list overflowed its arena
    makes every rank reopen with a larger one and repeat (the relations
    already merged are true ones, so a repeat is exact)."""

    def __init__(self, ctx, n: int, group=None, cap: int | None = None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.ctx = ctx
        self.n = n
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.cap = cap or max(1 << 16, n // 64)
        self.device = device  # device of the flag tensor (NCCL); None = CPU (gloo)
        self.reopens = 0
        self._connect()

    def _connect(self):
        # Every step is collective, so a rank that cannot open or map an
        # arena (no CUDA IPC between the processes, no peer access) makes all
        # ranks raise PeerUnavailable together instead of leaving the others
        # blocked in a collective: the caller can fall back to NCCL.
        err = ""
        try:
            blob = self.ctx.peer_open(self.n, self.cap, self.rank, self.world)
        except Exception as exc:  # noqa: BLE001 (any failure: same protocol)
            blob, err = b"", f"rank {self.rank}: {exc}"
        blobs = [None] * self.world
        self.dist.all_gather_object(blobs, blob, group=self.group)
        if not all(blobs):
            if blob:
                self.ctx.peer_close()
            raise PeerUnavailable(err or "a peer could not open its export arena")
        try:
            self.ctx.peer_connect(b"".join(blobs))
        except Exception as exc:  # noqa: BLE001
            err = f"rank {self.rank}: {exc}"
        if self._any(bool(err)):
            self.ctx.peer_disconnect()
            self.dist.barrier(group=self.group)
            self.ctx.peer_close()
            raise PeerUnavailable(err or "a peer could not map the export arenas")

    def _any(self, flag: bool) -> bool:
        import torch
        t = torch.tensor([int(flag)], dtype=torch.int32, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def merge(self, forest) -> dict:
        for attempt in range(3):
            self.ctx.peer_export(forest)
            self.dist.barrier(group=self.group)
            mx, overflow = self.ctx.peer_merge(forest)
            if not self._any(overflow):
                mx["reopens"] = self.reopens
                return mx
            self.cap = self.n if attempt >= 1 else min(self.n, 8 * self.cap)
            self.reopens += 1
            self._release()
            self._connect()
        raise RuntimeError("peer merge: pair arenas kept overflowing")

    def _release(self):
        # every rank unmaps its peers' arenas before any rank frees its own
        self.ctx.peer_disconnect()
        self.dist.barrier(group=self.group)

    def close(self):
        self._release()
        self.ctx.peer_close()


def merge_round_p2p(peer: PeerMerge, forest) -> MergeTimes:
    """export -> barrier -> NVLink gather + re-hook on this rank."""
    t = MergeTimes()
    t0 = time.perf_counter()
    mx = peer.merge(forest)
    t.rehook_ms = 1e3 * (time.perf_counter() - t0)
    t.extra = {"device_ms": mx["total_ms"], "reopens": mx["reopens"]}
    t.pairs_sent = int(mx["m"])
    t.pairs_received = int(mx["edges_processed"])
    t.bits_bytes = 4 * ((peer.n + 31) // 32)
    t.rehook_passes = int(mx["passes"])
    return t
