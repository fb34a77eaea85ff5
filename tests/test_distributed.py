"""Multi-GPU merge protocol — CPU (gloo, world_size 2 and 3)
and a one-GPU emulation of G ranks through the real kernels.

The CPU tests run the exact exchange code of paper_1612_01178_b200.distributed
over torch.distributed/gloo; only the per-rank compute (local CC, export,
re-hook) is played by a numpy stand-in built on the oracle, because there is
no GPU here.  The GPU emulation test runs the real export/re-hook kernels for
G logical ranks one after another on one device (no kernel waits on another).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_01178_b200.distributed import edge_range, exchange, merge_round, or_rows


def test_edge_range_matches_partition_edges(oracle):
    import ctypes as C
    for m, w in [(10, 3), (6, 1), (5, 5), (0, 4), (2**32, 8), (1000003, 7)]:
        firsts = [edge_range(m, w, r) for r in range(w)]
        assert sum(c for _, c in firsts) == m
        if m < 10**7:
            b = np.zeros(min(max(w, 1), max(m, 1)) + 1, dtype=np.uint64)
            cl = C.c_int()
            k = oracle._olib().oracle_partition(m, w, b.ctypes.data, C.byref(cl))
            if k == w:
                assert [f for f, _ in firsts] + [m] == b[: k + 1].tolist()


class NumpyBackend:
    """CPU stand-in for one rank (oracle-based; test-only)."""

    def __init__(self, oracle, n, shard):
        self.O, self.n, self.shard = oracle, n, shard
        self.pi = None

    def local_cc(self):
        self.pi = self.O.cc(self.n, self.shard).astype(np.int64)  # stars: pi(v) = label

    def export(self):
        n, pi = self.n, self.pi
        v = np.arange(n)
        in0 = (pi == 0) & (v != 0)
        words = np.zeros((n + 31) // 32, dtype=np.uint32)
        np.bitwise_or.at(words, v[in0] >> 5, (np.uint32(1) << (v[in0] & 31).astype(np.uint32)))
        keep = (pi != v) & (pi != 0)
        pairs = np.stack([v[keep], pi[keep]], 1).astype(np.int32)
        return torch.from_numpy(words.view(np.int32)), torch.from_numpy(pairs).reshape(-1, 2)

    def rehook(self, bits_or, remote):
        n = self.n
        words = bits_or.numpy().view(np.uint32)
        vs = np.nonzero(((words[np.arange(n) >> 5] >> (np.arange(n) & 31).astype(np.uint32)) & 1))[0]
        local = np.stack([np.arange(n), self.pi], 1)
        e = np.concatenate([local, np.stack([vs, np.zeros_like(vs)], 1),
                            remote.numpy().astype(np.int64).reshape(-1, 2)]).astype(np.uint64)
        self.pi = self.O.cc(n, e).astype(np.int64)
        return {"passes": 1}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        kind, n, e = spec
        first, count = edge_range(e.shape[0], world, rank)
        be = NumpyBackend(O, n, e[first:first + count])
        be.local_cc()
        t = merge_round(be)
        q.put((rank, be.pi.tolist(), t.pairs_sent, t.pairs_received))
        dist.destroy_process_group()
    except Exception as ex:  # surface errors to the parent
        q.put((rank, repr(ex), 0, 0))


def _graphs():
    import oracle as O
    return [("rmat", 1 << 12, O.gen_rmat(12, 8, 5)),
            ("er", 3000, O.gen_er(3000, 4000, 7)),
            ("grid", 40 * 37, O.gen_grid(40, 37))]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("gi", [0, 1, 2])
def test_gloo_merge_protocol(oracle, world, gi):
    spec = _graphs()[gi]
    want = oracle.cc(spec[1], spec[2]).astype(np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, q)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=180) for _ in range(world)]
    [p.join(timeout=60) for p in procs]
    for rank, labels, sent, recv in res:
        assert not isinstance(labels, str), labels
        assert np.array_equal(np.asarray(labels), want), (spec[0], world, rank)


def test_exchange_single_rank():
    """world = 1: nothing remote, empty payloads pass through."""
    port = _free_port()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        bits = torch.tensor([5, 0, 7], dtype=torch.int32)
        pairs = torch.tensor([[3, 1]], dtype=torch.int32)
        rows, rank, p = exchange(bits, pairs)
        assert rank == 0 and rows.tolist() == [[5, 0, 7]] and p.shape == (0, 2)
        assert or_rows(rows, rank).tolist() == [0, 0, 0]
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ one-GPU emulation

@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("spec", ["rmatx:scale=18,ef=16,seed=3", "erx:n=200000,m=1000000,seed=2",
                                  "grid:300x301"])
def test_gpu_emulated_ranks(ctx, oracle, G, spec):
    """G logical ranks on one GPU, sequentially: the real local CC, export and
    re-hook kernels, the exchange done in-process (OR of the other ranks'
    bitmaps, concatenation of their pairs)."""
    full = ctx.generate(spec)
    n, m = full.n, full.m
    want = oracle.cc(n, full.edges()).astype(np.uint64)
    dev = torch.device("cuda:0")
    from paper_1612_01178_b200.distributed import CudaBackend
    ranks = []
    for r in range(G):
        first, count = edge_range(m, G, r)
        g = ctx.generate_range(spec, first, count)
        be = CudaBackend(ctx, n, dev)
        be.local_cc(g)
        bits, pairs = be.export()
        ranks.append((be, bits.clone(), pairs.clone()))
    # the gathered bitmap rows as NCCL would lay them out (row stride
    # send_offset(nwords) + 2, the pair count in the tail words)
    from paper_1612_01178_b200.distributed import send_offset
    nw = ranks[0][1].numel()
    rows = torch.zeros((G, send_offset(nw) + 2), dtype=torch.int32, device=dev)
    for s, (_, b, _) in enumerate(ranks):
        rows[s, :nw] = b
    for r, (be, _, _) in enumerate(ranks):
        remote = torch.cat([p for s, (_, _, p) in enumerate(ranks) if s != r])
        if r % 2:
            # row-aware re-hook: the kernel ORs every row but r's
            be.rehook_rows(rows[:, :nw], r, remote)
        else:
            bits_or = torch.zeros_like(ranks[0][1])
            for s, (_, b, _) in enumerate(ranks):
                if s != r:
                    bits_or |= b
            be.rehook(bits_or, remote)
        assert np.array_equal(be.labels(), want), (spec, G, r)
