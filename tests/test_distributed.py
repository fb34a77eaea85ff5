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
from pathlib import Path

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


# ------------------------------------------------------- CUDA-IPC merge protocol

class FakePeerCtx:
    """CPU stand-in for the hcc_peer_* entry points (test-only): the "arena"
    of a rank is a file in a shared directory, the handle blob is its path.
    Export truncates the pair list at the arena's capacity but records the
    full count, like k_export; merge reads every peer's file (the IPC read)
    and re-hooks with the oracle."""

    def __init__(self, oracle, n, shard, root):
        self.O, self.n, self.root = oracle, n, root
        self.pi = oracle.cc(n, shard).astype(np.int64)
        self.opens = 0

    def peer_open(self, n, cap, rank, world):
        self.cap, self.rank, self.world = cap, rank, world
        self.opens += 1
        self.path = os.path.join(self.root, f"arena{rank}.{self.opens}.npz")
        return self.path.encode().ljust(256, b"\0")

    def peer_connect(self, handles):
        self.peers = [handles[i * 256:(i + 1) * 256].rstrip(b"\0").decode()
                      for i in range(self.world)]

    def peer_export(self, forest):
        v = np.arange(self.n)
        keep = (self.pi != v) & (self.pi != 0)
        pairs = np.stack([v[keep], self.pi[keep]], 1)
        np.savez(self.path, in0=v[(self.pi == 0) & (v != 0)], pairs=pairs[: self.cap],
                 count=len(pairs), cap=self.cap)

    def peer_merge(self, forest):
        rels, overflow = [np.stack([np.arange(self.n), self.pi], 1)], False
        for r, path in enumerate(self.peers):
            d = np.load(path)
            overflow |= int(d["count"]) > int(d["cap"])
            if r != self.rank:
                rels.append(np.stack([d["in0"], np.zeros_like(d["in0"])], 1))
                rels.append(d["pairs"].reshape(-1, 2))
        self.pi = self.O.cc(self.n, np.concatenate(rels).astype(np.uint64)).astype(np.int64)
        return {"total_ms": 0.0, "m": 0, "edges_processed": 0, "passes": 1}, overflow

    def peer_disconnect(self):
        pass

    def peer_close(self):
        pass


def _peer_worker(rank, world, port, spec, root, cap, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from paper_1612_01178_b200.distributed import PeerMerge
        kind, n, e = spec
        first, count = edge_range(e.shape[0], world, rank)
        fc = FakePeerCtx(O, n, e[first:first + count], root)
        pm = PeerMerge(fc, n, cap=cap)
        pm.merge(None)
        q.put((rank, fc.pi.tolist(), pm.reopens))
        dist.destroy_process_group()
    except Exception as ex:  # surface errors to the parent
        q.put((rank, repr(ex), 0))


@pytest.mark.parametrize("world,gi,cap", [(2, 0, None), (3, 1, None), (2, 2, 4), (3, 0, 1)])
def test_gloo_peer_merge_protocol(oracle, tmp_path, world, gi, cap):
    """PeerMerge (the CUDA-IPC transport's host protocol: handle all-gather,
    export -> barrier -> merge -> overflow all-reduce, reopen on overflow),
    world 2 and 3 over gloo; tiny caps force the reopen path."""
    spec = _graphs()[gi]
    want = oracle.cc(spec[1], spec[2]).astype(np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, spec, str(tmp_path), cap, q))
             for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=180) for _ in range(world)]
    [p.join(timeout=60) for p in procs]
    for rank, labels, reopens in res:
        assert not isinstance(labels, str), labels
        assert np.array_equal(np.asarray(labels), want), (spec[0], world, rank)
        if cap is not None:
            assert reopens >= 1


class _FailingPeerCtx(FakePeerCtx):
    def __init__(self, *a, fail_rank=0, fail_at="connect", **k):
        super().__init__(*a, **k)
        self.fail_rank, self.fail_at = fail_rank, fail_at
        self.closed = self.disconnected = 0

    def peer_open(self, n, cap, rank, world):
        if self.fail_at == "open" and rank == self.fail_rank:
            raise RuntimeError("no CUDA IPC (test)")
        return super().peer_open(n, cap, rank, world)

    def peer_connect(self, handles):
        if self.fail_at == "connect" and self.rank == self.fail_rank:
            raise RuntimeError("cudaIpcOpenMemHandle failed (test)")
        super().peer_connect(handles)

    def peer_disconnect(self):
        self.disconnected += 1

    def peer_close(self):
        self.closed += 1


def _unavailable_worker(rank, world, port, spec, root, fail_at, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from paper_1612_01178_b200.distributed import PeerMerge, PeerUnavailable
        kind, n, e = spec
        first, count = edge_range(e.shape[0], world, rank)
        fc = _FailingPeerCtx(O, n, e[first:first + count], root, fail_rank=world - 1,
                             fail_at=fail_at)
        try:
            PeerMerge(fc, n)
            q.put((rank, "connected"))
        except PeerUnavailable:
            q.put((rank, f"unavailable closed={fc.closed}"))
        dist.destroy_process_group()
    except Exception as ex:  # surface errors to the parent
        q.put((rank, repr(ex)))


@pytest.mark.parametrize("world,fail_at", [(2, "open"), (3, "open"), (2, "connect"),
                                           (3, "connect")])
def test_gloo_peer_merge_unavailable_everywhere(oracle, tmp_path, world, fail_at):
    """One rank cannot open or map the CUDA-IPC arenas: every rank raises
    PeerUnavailable together (no rank is left blocked in a collective) and
    releases what it opened, so bench.py can fall back to the NCCL merge."""
    spec = _graphs()[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unavailable_worker,
                         args=(r, world, port, spec, str(tmp_path), fail_at, q))
             for r in range(world)]
    [p.start() for p in procs]
    res = dict(q.get(timeout=180) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    for rank in range(world):
        msg = res[rank]
        assert msg.startswith("unavailable"), (rank, msg)
        failed_open = fail_at == "open" and rank == world - 1
        assert msg.endswith("closed=0" if failed_open else "closed=1"), (rank, msg)


@pytest.mark.gpu
@pytest.mark.parametrize("world,cap", [(2, 0), (3, 0), (2, 16)])
def test_gpu_ipc_merge_multiprocess(oracle, tmp_path, world, cap):
    """The CUDA-IPC transport end to end: `world` processes (torchrun, gloo
    for the host collectives) share device 0, map each other's export arenas
    and merge with k_merge_gather; every rank's labels equal the oracle's.
    cap=16 forces the overflow -> reopen path.  Several runs per process
    exercise the arena reuse between runs."""
    import hashlib
    import json
    import subprocess
    import sys
    spec = "rmatx:scale=16,ef=16,seed=5"
    e = oracle.gen_rmatx(16, 5, 0, 16 << 16)
    want = oracle.cc(1 << 16, e).astype(np.uint32)
    out = tmp_path / "res"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={_free_port()}",
                        str(Path(__file__).parent / "ipc_worker.py"), spec, str(out), str(cap), "3"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    for rank in range(world):
        res = json.loads(Path(f"{out}.{rank}").read_text())
        assert res["sha"] == hashlib.sha256(want.tobytes()).hexdigest(), res
        assert res["components"] == int(np.sum(want == np.arange(1 << 16, dtype=np.uint32)))
        if cap:
            assert res["reopens"] >= 1


@pytest.mark.gpu
def test_bench_multi_rank_path_on_one_gpu(tmp_path):
    """bench.py's N > 1 code path (torchrun, 2 ranks; --share-gpus puts both
    on the one GPU of the test box and uses gloo for the host collectives):
    edge-partitioned RMAT-24, local CC + CUDA-IPC merge, e2e leg, the
    reference-arm rule (rank 0 alone).  Checks the JSON line's schema and
    that both ranks hold the same, correct labels."""
    import json
    import subprocess
    import sys
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(root / "bench.py"),
           "--gpus", "2", "--share-gpus", "--workload", "rmat24", "--steps", "2",
           "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["labels_consistent_across_ranks"] and d["components"] == 7908545
    assert d["config"]["edges_per_gpu"] == (1 << 27)
    for k in ("roofline", "e2e", "clocks", "merge", "timing"):
        assert k in d
    assert d["e2e"]["value"] > 0 and d["merge"]["reopens"] == 0
