"""Parity of the CUDA path (through the C-ABI) against the oracle and the
reference's golden vectors.  Bit-exact: labels are integers.

Mirrors the reference suites: test_forest.cpp (kernel KATs, stress,
monotonicity), test_engines.cpp (engine KATs, segment invariance, algorithm
agreement, schedule independence, observer invariants, per-segment metrics),
acceptance.cpp C1/C2/C4/C5/C6, test_generators.cpp and test_oracle.cpp.
"""
from __future__ import annotations

import json
import threading
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
ALGOS = ["baseline", "baseline-mj", "atomic", "adaptive"]


def digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def run(ctx, n, edges, algo, **kw):
    g = ctx.graph_from_edges(np.asarray(edges, dtype=np.uint64).reshape(-1, 2), n)
    lab, mx = ctx.cc(g, algo, **kw)
    g.close()
    return lab.astype(np.uint64), mx


# --------------------------------------------------------------- forest KATs

def forest(ctx, parents):
    f = ctx.forest(len(parents))
    if len(parents):
        f.upload(parents)
    return f


def test_forest_init(ctx):  # test_forest.cpp:33-37
    assert ctx.forest(5).snapshot().tolist() == [0, 1, 2, 3, 4]
    assert ctx.forest(0).snapshot().tolist() == []
    assert ctx.forest(1).snapshot().tolist() == [0]


def test_forest_hook_jump(ctx):  # test_forest.cpp:39-63
    f = ctx.forest(3)
    assert f.hook(0, 2) and f.snapshot().tolist() == [0, 1, 0]
    f = forest(ctx, [0, 0, 2])
    assert f.hook(1, 2) and f.snapshot().tolist() == [0, 0, 0]
    f = forest(ctx, [0, 0, 1])
    assert not f.hook(1, 1) and f.snapshot().tolist() == [0, 0, 1]
    f = forest(ctx, [0, 0, 1])
    assert f.jump(2) and f.snapshot().tolist() == [0, 0, 0]
    assert not f.jump(2)
    assert not ctx.forest(1).jump(0)


def test_forest_atomic_hook(ctx, capi):  # test_forest.cpp:65-114
    f = ctx.forest(5)
    c = capi.Counters()
    f.atomic_hook(2, 4, c)
    assert f.snapshot().tolist() == [0, 1, 2, 3, 2]
    assert (c.hook_traversal_steps, c.cas_failures) == (1, 0)
    f = forest(ctx, [0, 1, 0, 1])
    f.atomic_hook(2, 3, capi.Counters())
    assert f.snapshot().tolist() == [0, 0, 0, 1]
    f = forest(ctx, [0, 0, 0])
    c = capi.Counters()
    f.atomic_hook(1, 2, c)
    assert f.snapshot().tolist() == [0, 0, 0] and c.hook_traversal_steps == 0
    for depth in [1, 2, 17, 1024]:
        f = forest(ctx, [0] + list(range(depth)))
        c = capi.Counters()
        f.atomic_hook(depth, 0, c)
        assert c.hook_traversal_steps <= depth + 1


def test_forest_atomic_hook_random(ctx, capi, oracle):  # test_forest.cpp:91-105
    rng = np.random.default_rng(11)
    for _ in range(60):
        n = int(2 + rng.integers(0, 30))
        pi = [0] + [int(rng.integers(0, v + 1)) for v in range(1, n)]
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        f = forest(ctx, pi)
        c = capi.Counters()
        f.atomic_hook(u, v, c)
        got = f.snapshot()
        # sequential device semantics equal the oracle's exactly
        want = np.asarray(pi, dtype=np.uint64)
        oc = np.zeros(3, dtype=np.uint64)
        oracle._olib().oracle_atomic_hook(want.ctypes.data, u, v, oc.ctypes.data)
        assert np.array_equal(got, want)
        assert (c.hook_traversal_steps, c.cas_failures) == (oc[0], oc[1])


def test_forest_multi_jump(ctx, capi):  # test_forest.cpp:116-169, acceptance C5
    f = forest(ctx, [0, 0, 1, 2])
    c = capi.Counters()
    f.multi_jump(3, c)
    assert f.load(3) == 0 and c.jump_steps == 2
    f = forest(ctx, [0, 0])
    c = capi.Counters()
    f.multi_jump(1, c)
    assert c.jump_steps == 0
    k = 1000
    f = forest(ctx, [0] + list(range(k)))
    up = capi.Counters()
    f.multi_jump_range(0, k + 1, False, up)
    assert up.jump_steps == k - 1 and f.is_star()
    f = forest(ctx, [0] + list(range(k)))
    down = capi.Counters()
    f.multi_jump_range(0, k + 1, True, down)
    assert down.jump_steps == k * (k - 1) // 2 and f.is_star()
    # per-element calls, ascending, as the reference test loops
    f = forest(ctx, [0] + list(range(200)))
    c = capi.Counters()
    for v in range(201):
        f.multi_jump(v, c)
    assert c.jump_steps == 199


def test_forest_is_star_cas(ctx):  # test_forest.cpp:171-175; forest.hpp:39-43
    assert forest(ctx, [0, 0, 0, 3, 3]).is_star()
    assert not forest(ctx, [0, 0, 1]).is_star()
    assert ctx.forest(0).is_star()
    f = ctx.forest(4)
    ok, seen = f.cas(3, 3, 1)
    assert ok and f.load(3) == 1
    ok, seen = f.cas(3, 3, 0)
    assert not ok and seen == 1


def test_forest_concurrent_stress(ctx, capi):  # test_forest.cpp:185-211
    n = 2000
    rng = np.random.default_rng(7)
    edges = rng.integers(0, n, size=(6000, 2))
    f = ctx.forest(n)
    errors = []

    def worker(seed):
        try:
            r = np.random.default_rng(seed)
            c = capi.Counters()
            for _ in range(1500):
                u, v = (int(x) for x in edges[r.integers(0, len(edges))])
                op = int(r.integers(0, 4))
                if op == 0:
                    f.hook(u, v)
                elif op == 1:
                    f.atomic_hook(u, v, c)
                elif op == 2:
                    f.jump(int(r.integers(0, n)))
                else:
                    f.multi_jump(int(r.integers(0, n)), c)
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(100 + t,)) for t in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errors
    snap = f.snapshot()
    assert np.all(snap <= np.arange(n, dtype=np.uint64))
    assert f.bound_ok()


def test_forest_monotonicity(ctx, capi):  # test_forest.cpp:213-229
    rng = np.random.default_rng(21)
    n = 64
    f = ctx.forest(n)
    prev = f.snapshot()
    for _ in range(300):
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        if rng.integers(0, 2):
            f.atomic_hook(u, v, capi.Counters())
        else:
            f.multi_jump(u, capi.Counters())
        cur = f.snapshot()
        assert np.all(cur <= prev)
        prev = cur


# --------------------------------------------------------------- engine KATs

@pytest.mark.parametrize("algo", ALGOS)
def test_engine_spec_examples(ctx, algo):  # test_engines.cpp:109-134
    assert run(ctx, 5, [(0, 1), (1, 2), (3, 4)], algo)[0].tolist() == [0, 0, 0, 3, 3]
    assert run(ctx, 4, np.zeros((0, 2)), algo)[0].tolist() == [0, 1, 2, 3]
    k4 = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    assert run(ctx, 4, k4, algo)[0].tolist() == [0, 0, 0, 0]
    assert run(ctx, 6, [(0, 5)], algo)[0].tolist() == [0, 1, 2, 3, 4, 0]
    assert run(ctx, 3, [(1, 2)], algo, segments=1)[0].tolist() == [0, 1, 1]
    lab, mx = run(ctx, 0, np.zeros((0, 2)), algo)
    assert lab.tolist() == [] and mx["components"] == 0


def test_adaptive_auto_s_on_grid(ctx, oracle):  # test_engines.cpp:127-131, test_bench.cpp:30-41
    lab, mx = run(ctx, 4, oracle.gen_grid(2, 2), "adaptive", segments=0)
    assert mx["s"] == 2 and lab.tolist() == [0, 0, 0, 0]
    lab, mx = run(ctx, 900, oracle.gen_grid(30, 30), "adaptive", segments=0)
    assert mx["s"] == 4 and mx["components"] == 1


def test_segments_clamped(ctx):  # test_bench.cpp:126-134, engines.hpp:43-50
    lab, mx = run(ctx, 4, [(0, 1), (2, 3)], "adaptive", segments=50)
    assert mx["s"] == 2 and mx["segments_clamped"] and lab.tolist() == [0, 0, 2, 2]


def test_exhaustive_small_graphs(ctx, oracle):  # acceptance.cpp:51-73 (C1)
    rng = np.random.default_rng(20260824)
    for _ in range(250):
        n = int(rng.integers(1, 9))
        e = rng.integers(0, n, size=(int(rng.integers(0, 14)), 2)).astype(np.uint64)
        want = oracle.bfs_cc(n, e)
        g = ctx.graph_from_edges(e, n)
        for algo in ALGOS:
            for s in ([1, 2, 0, max(1, len(e))] if algo == "adaptive" else [0]):
                lab, _ = ctx.cc(g, algo, segments=s)
                assert np.array_equal(lab.astype(np.uint64), want), (algo, s, e.tolist())
        g.close()


def test_segment_count_invariance(ctx, oracle):  # test_engines.cpp:136-149
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(1, 61))
        e = rng.integers(0, n, size=(int(rng.integers(0, 120)), 2)).astype(np.uint64)
        want = oracle.cc(n, e)
        g = ctx.graph_from_edges(e, n)
        m = max(1, len(e))
        for s in [1, 2, 4, 8, m, 0]:
            assert np.array_equal(ctx.cc(g, "adaptive", segments=s)[0], want)
            assert np.array_equal(ctx.cc(g, "baseline-mj", first_pass_segments=s)[0], want)
        g.close()


FAMILIES = ["er", "rmat", "grid"]


@pytest.mark.parametrize("family", FAMILIES)
def test_random_families(ctx, oracle, family):  # acceptance.cpp:77-122 (C2)
    rng = np.random.default_rng({"er": 1, "rmat": 2, "grid": 3}[family])
    for i in range(40):
        if family == "er":
            n = int(rng.integers(1, 4097))
            e = oracle.gen_er(n, int(rng.integers(0, 4 * n + 1)), int(rng.integers(0, 2**63)))
        elif family == "rmat":
            sc = int(rng.integers(4, 13))
            n = 1 << sc
            e = oracle.gen_rmat(sc, int(rng.integers(1, 17)), int(rng.integers(0, 2**63)))
        else:
            r, c = int(rng.integers(1, 65)), int(rng.integers(1, 65))
            n, e = r * c, oracle.gen_grid(r, c)
        want = oracle.cc(n, e)
        g = ctx.graph_from_edges(e, n)
        for algo in ALGOS:
            lab, mx = ctx.cc(g, algo, max_threads=[0, 4, 1][i % 3] if algo != "baseline" else 0)
            assert np.array_equal(lab.astype(np.uint64), want), (family, i, algo)
            assert mx["components"] == int(np.sum(want == np.arange(n)))
        g.close()


@pytest.mark.parametrize("algo", ALGOS)
def test_phase_observer_invariants(ctx, oracle, algo):  # test_engines.cpp:189-208
    rng = np.random.default_rng(10)
    for _ in range(6):
        n = int(rng.integers(1, 201))
        e = rng.integers(0, n, size=(int(rng.integers(0, 500)), 2)).astype(np.uint64)
        g = ctx.graph_from_edges(e, n)
        seen = {"compress": 0}

        def obs(phase, f):
            snap = f.snapshot()
            assert np.all(snap <= np.arange(n, dtype=np.uint64))
            if phase == 1:
                assert f.is_star()
                seen["compress"] += 1

        lab, mx = ctx.cc(g, algo, segments=3, first_pass_segments=3, observer=obs)
        assert np.array_equal(lab, oracle.cc(n, e).astype(np.uint32))
        if algo == "adaptive":
            assert seen["compress"] == mx["s"]
        g.close()


def test_algorithm_agreement_and_flags(ctx, oracle, capi):  # test_engines.cpp:151-177
    rng = np.random.default_rng(6)
    for _ in range(20):
        n = int(rng.integers(1, 61))
        e = rng.integers(0, n, size=(int(rng.integers(0, 120)), 2)).astype(np.uint64)
        want = oracle.bfs_cc(n, e)
        g = ctx.graph_from_edges(e, n)
        for fl in [0, capi.FLAG_FULL_PASSES, capi.FLAG_HOST_LOOP, capi.FLAG_NO_GRAPH,
                   capi.FLAG_CHECK_STAR]:
            assert np.array_equal(ctx.cc(g, "baseline-mj", flags=fl)[0].astype(np.uint64), want)
        g.close()
    # schedule independence: thread caps and edge shuffles
    e = oracle.gen_er(300, 600, 17)
    want = oracle.cc(300, e)
    for mt in [1, 2, 4, 0]:
        assert np.array_equal(run(ctx, 300, e, "adaptive", segments=4, max_threads=mt)[0], want)
        assert np.array_equal(run(ctx, 300, e, "baseline", max_threads=mt)[0], want)
    for _ in range(5):
        e = rng.permutation(e)
        assert np.array_equal(run(ctx, 300, e, "adaptive", segments=4)[0], want)


def test_baseline_outer_iteration_cap(ctx):  # test_engines.cpp:179-187
    rng = np.random.default_rng(9)
    for _ in range(10):
        n = int(rng.integers(1, 501))
        e = rng.integers(0, n, size=(int(rng.integers(0, 2000)), 2))
        _, mx = run(ctx, n, e, "baseline")
        assert mx["outer_iterations"] <= 4 * np.ceil(np.log2(n + 2)) + 2


def test_single_thread_determinism(ctx, oracle):  # test_engines.cpp:210-220
    e = oracle.gen_rmat(8, 8, 23)
    a = run(ctx, 256, e, "adaptive", segments=0, max_threads=1)[1]
    b = run(ctx, 256, e, "adaptive", segments=0, max_threads=1)[1]
    for k in ("hook_traversal_steps", "cas_failures", "jump_steps", "s"):
        assert a[k] == b[k]


def test_per_segment_metrics_sum(ctx, oracle):  # test_engines.cpp:222-232
    e = oracle.gen_er(500, 3000, 31)
    g = ctx.graph_from_edges(e, 500)
    _, mx = ctx.cc(g, "adaptive", segments=5)
    segs = ctx.segments()
    assert len(segs) == mx["s"] == 5
    for k in ("hook_traversal_steps", "cas_failures", "jump_steps"):
        assert sum(s[k] for s in segs) == mx[k]
    g.close()


# ----------------------------------------------------- golden (reference) vectors

def _golden_graph(oracle, name):
    gold = GOLD["graphs"][name]
    if "edges" in gold:
        e = np.asarray(gold["edges"], dtype=np.uint64).reshape(-1, 2)
    elif name.startswith("rmat"):
        sc, ef, s = (int(x.lstrip("efs")) for x in name[4:].split("_"))
        e = oracle.gen_rmat(sc, ef, s)
    elif name.startswith("grid"):
        r, c = (int(x) for x in name[4:].split("x"))
        e = oracle.gen_grid(r, c)
    else:
        n, m, s = name[2:].split("_")
        e = oracle.gen_er(int(n), int(m), int(s[1:]))
    assert digest(e) == gold["edges_sha256"]
    return gold["n"], e


@pytest.mark.parametrize("name", sorted(GOLD["graphs"]))
def test_golden_labels_and_counters(ctx, oracle, name):
    gold = GOLD["graphs"][name]
    n, e = _golden_graph(oracle, name)
    g = ctx.graph_from_edges(e, n)
    for algo in ALGOS:
        lab, mx = ctx.cc(g, algo)
        assert digest(lab.astype(np.uint64)) == gold["labels_sha256"], algo
        assert mx["components"] == gold["components"]
    st = g.stats()
    assert st["m_unique"] == gold["stats"]["m_unique"]
    assert st["max_degree"] == gold["stats"]["max_degree"]
    assert st["avg_degree"] == gold["stats"]["avg_degree"]
    # One device thread executes the reference's workers = 1 schedule, so the
    # work counters equal the reference's exactly.
    for key, want in gold["engines"].items():
        if key == "baseline-mj":
            lab, mx = ctx.cc(g, "baseline-mj", max_threads=1, flags=1)  # literal full passes
        elif key == "baseline":
            lab, mx = ctx.cc(g, "baseline", max_threads=1)
        elif key == "atomic":
            lab, mx = ctx.cc(g, "atomic", max_threads=1)
        else:
            lab, mx = ctx.cc(g, "adaptive", segments=int(key.split("_s")[1]), max_threads=1)
        assert digest(lab.astype(np.uint64)) == gold["labels_sha256"], key
        for k in ("s", "outer_iterations", "jump_steps", "cas_failures", "hook_traversal_steps"):
            assert mx[k] == want[k], (key, k, mx[k], want[k])
        if want.get("segment_counters"):
            segs = ctx.segments()
            got = [[s["hook_traversal_steps"], s["cas_failures"], s["jump_steps"]] for s in segs]
            assert got[:len(want["segment_counters"])] == want["segment_counters"], key
    g.close()


# ------------------------------------------------------------- ingestion / gens

def test_device_generators_match_oracle_twins(ctx, oracle):
    g = ctx.generate("rmatx:scale=14,ef=16,seed=3")
    assert np.array_equal(g.edges(), oracle.gen_rmatx(14, 3, 0, g.m))
    assert g.checksum() == oracle.checksum_u32(g.edges())
    g = ctx.generate("rmatx:scale=10,ef=4,seed=9,a=0.45,b=0.25,c=0.15,d=0.15")
    assert np.array_equal(g.edges(), oracle.gen_rmatx(10, 9, 0, g.m, a=0.45, b=0.25, c=0.15))
    g = ctx.generate("erx:n=100000,m=300000,seed=4")
    assert np.array_equal(g.edges(), oracle.gen_erx(100000, 4, 0, 300000))
    g = ctx.generate("grid:37x53")
    assert np.array_equal(g.edges().astype(np.uint64), oracle.gen_grid(37, 53))
    g = ctx.generate("rmatx:scale=8,ef=8", default_seed=23)
    assert np.array_equal(g.edges(), oracle.gen_rmatx(8, 23, 0, g.m))


def test_generator_errors(ctx, capi):
    for spec in ["wat:1", "erx:n=10", "grid", "grid:0x3", "erx:n=0,m=3",
                 "rmatx:scale=4,ef=2,a=0.5,b=0.3,c=0.3,d=0.3"]:
        with pytest.raises(capi.HccError) as ei:
            ctx.generate(spec)
        assert ei.value.code == capi.HCC_EINVAL


def test_csr_ingestion(ctx, oracle):
    rng = np.random.default_rng(3)
    n = 3000
    e = rng.integers(0, n, size=(9000, 2))
    order = np.lexsort((e[:, 1], e[:, 0]))
    e = e[order]
    rp = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(rp, e[:, 0] + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    g = ctx.graph_from_csr(rp, e[:, 1].astype(np.uint32))
    assert np.array_equal(g.edges().astype(np.int64), e)
    assert np.array_equal(ctx.cc(g)[0], oracle.cc(n, e.astype(np.uint64)).astype(np.uint32))


def test_ingestion_errors(ctx, capi):
    with pytest.raises(capi.HccError) as ei:
        ctx.graph_from_edges(np.array([[0, 5]], dtype=np.uint64), 5)
    assert ei.value.code == capi.HCC_ERANGE
    with pytest.raises(capi.HccError) as ei:
        ctx.graph_from_edges(np.array([[0, 5]], dtype=np.uint32), 5)
    assert ei.value.code == capi.HCC_ERANGE
    with pytest.raises(capi.HccError) as ei:
        ctx.graph_from_edges(np.zeros((0, 2), dtype=np.uint64), 1 << 32)
    assert ei.value.code == capi.HCC_EINVAL
    g = ctx.graph_from_edges(np.array([[0, 1]], dtype=np.uint64), 3)
    f = ctx.forest(4)
    with pytest.raises(capi.HccError):
        ctx.cc(g, forest=f)


def test_in_place_forest(ctx, oracle):  # *_cc_into contract (engines.hpp:183-231)
    e = oracle.gen_rmat(10, 8, 4)
    n = 1024
    g = ctx.graph_from_edges(e, n)
    f = ctx.forest(n)
    f.upload(np.zeros(n, dtype=np.uint64))  # garbage-in: reset inside
    for algo in ALGOS:
        lab, _ = ctx.cc(g, algo, forest=f)
        assert np.array_equal(f.snapshot(), oracle.cc(n, e))
        assert f.is_star()


@pytest.mark.parametrize("spec", ["rmatx:scale=20,ef=16,seed=7", "erx:n=1100000,m=9000000,seed=3",
                                  "erx:n=1048579,m=8000000,seed=5", "erx:n=70001,m=40000,seed=9",
                                  "grid:1100x1000"])
def test_star0_bitmap_paths(ctx, oracle, spec):
    """The star-0 bitmap fast path (n >= 2^16) and the plain gather path give
    identical labels under every topology plan."""
    import os
    g = ctx.generate(spec)
    want = oracle.cc(g.n, g.edges())
    for s0b, walk in [("1", "32"), ("0", "32"), ("1", "2"), ("1", "1"), ("0", "1")]:
        # (HCC_S0B_MIN_LOG2: the bitmap below its default n = 2^20 floor too)
        os.environ.update(HCC_S0B=s0b, HCC_WALK=walk, HCC_S0B_MIN_LOG2="16")
        try:
            for fps in [0, 1, 3]:
                lab, mx = ctx.cc(g, "baseline-mj", first_pass_segments=fps)
                assert np.array_equal(lab, want), (spec, s0b, walk, fps)
                assert mx["star0_bitmap"] == (s0b == "1")
        finally:
            for k in ("HCC_S0B", "HCC_WALK", "HCC_S0B_MIN_LOG2"):
                os.environ.pop(k, None)


def test_degenerate_graphs_with_star_machinery(ctx, oracle):
    """n >= 2^16 turns on the star bitmap, summary, sampler and chunked
    appends: empty, single-edge, self-loop-only and boundary-vertex graphs."""
    n = 70001  # not a multiple of 32: partial last bitmap / summary words
    rng = np.random.default_rng(5)
    cases = {
        "empty": np.zeros((0, 2), np.uint64),
        "one": np.array([[n - 1, 0]], np.uint64),
        "loops": np.repeat(np.arange(0, n, 7, dtype=np.uint64)[:, None], 2, axis=1),
        "last": np.stack([np.full(5000, n - 1, np.uint64),
                          rng.integers(0, n, 5000).astype(np.uint64)], axis=1),
        "path_rev": np.stack([np.arange(n - 1, 0, -1, dtype=np.uint64),
                              np.arange(n - 2, -1, -1, dtype=np.uint64)], axis=1),
    }
    import os
    os.environ["HCC_S0B_MIN_LOG2"] = "16"  # (the worklist engine's bitmap too)
    try:
        for name, e in cases.items():
            want = oracle.cc(n, e)
            for algo in ALGOS:
                lab, mx = run(ctx, n, e, algo)
                assert np.array_equal(lab, want.astype(np.uint64)), (name, algo)
                assert mx["components"] == int(np.sum(want == np.arange(n, dtype=np.uint32)))
    finally:
        os.environ.pop("HCC_S0B_MIN_LOG2", None)


@pytest.mark.parametrize("shift", [1, 977])
def test_star_moves_off_vertex0(ctx, oracle, shift):
    """Vertex 0 isolated (ER endpoints shifted by `shift`): the star bitmap must
    follow the giant component's root (sampled on the device) and give the
    oracle's labels under every plan, with and without the summary hook."""
    import os
    n = 1 << 21
    e = oracle.gen_erx(n - shift, 5, 0, 12 * n).astype(np.uint64) + shift
    g = ctx.graph_from_edges(e.astype(np.uint32), n)
    want = oracle.cc(n, e)
    assert want[0] == 0 and np.sum(want == 0) == 1  # vertex 0 alone
    for s0f in ("1", "0"):
        os.environ["HCC_S0F"] = s0f
        try:
            for plan in ("adapt:7:4", "adapt:9:4", "adapt:5:3"):
                os.environ["HCC_PLAN"] = plan
                lab, mx = ctx.cc(g, "baseline-mj")
                assert np.array_equal(lab, want), (s0f, plan)
        finally:
            os.environ.pop("HCC_PLAN", None)
            os.environ.pop("HCC_S0F", None)
    g.close()


def test_hook_events_flag_and_timeline(ctx, oracle, capi):
    """HCC_FLAG_HOOK_EVENTS adds per-launch CUDA events (bench roofline) without
    changing results; the device timeline is ordered hook -> compress -> next."""
    g = ctx.generate("rmatx:scale=20,ef=16,seed=3")
    want = oracle.cc(g.n, g.edges())
    for flags in (0, capi.FLAG_HOOK_EVENTS):
        lab, mx = ctx.cc(g, "baseline-mj", flags=flags)
        assert np.array_equal(lab, want)
        segs = ctx.segments()
        used = [s for s in segs[:mx["s"]] if s["edges_in"] > 0]
        assert used
        for s in used:
            assert (s["hook_event_ms"] >= 0) == bool(flags)
        prev = 0.0
        for s in segs:
            if s["hook_start_ms"] < 0:
                continue
            assert prev <= s["hook_start_ms"] <= s["hook_end_ms"], segs
            prev = s["hook_end_ms"]
            if s["compress_start_ms"] >= 0:
                assert s["hook_end_ms"] <= s["compress_start_ms"] <= s["compress_end_ms"]
                prev = s["compress_end_ms"]
        assert prev <= mx["total_ms"] + 0.05
        # each record names the hook kernel that ran its pass
        kinds = [s["hook_kernel"] for s in segs]
        assert kinds[0] in ("k_hook_small", "k_hook")
        assert all(k in ("k_hook_small", "k_hook", "k_hook_sum", "k_hook_sumd")
                   for k in kinds[1:mx["s"]])
        assert all(k == "k_hook_cas" for k in kinds[mx["s"]:])
    g.close()


def test_graph_assign_reuses_handle(ctx, oracle):
    """hcc_graph_assign_edges_u32 refills a handle; results track the new edges
    and the out-of-range check still applies."""
    a = oracle.gen_rmat(12, 8, 1).astype(np.uint32)
    b = oracle.gen_rmat(12, 8, 2).astype(np.uint32)
    g = ctx.graph_from_edges(a, 4096)
    assert np.array_equal(ctx.cc(g)[0], oracle.cc(4096, a))
    g.assign(b)
    assert np.array_equal(ctx.cc(g)[0], oracle.cc(4096, b))
    g.assign(a[:100], first=5)
    want = b.copy()
    want[5:105] = a[:100]
    assert np.array_equal(g.edges(), want)
    assert np.array_equal(ctx.cc(g)[0], oracle.cc(4096, want))
    import paper_1612_01178_b200.capi as C
    with pytest.raises(C.HccError) as ei:
        g.assign(np.array([[0, 4096]], dtype=np.uint32))
    assert ei.value.code == C.HCC_ERANGE


def test_async_upload_pipelined(ctx, oracle, capi):
    """hcc_graph_upload_async: two graph handles used alternately (the next
    input uploads on the copy stream while the current one runs, as the
    bench's pipelined e2e leg does) give the oracle's labels for each input;
    an out-of-range endpoint surfaces as HCC_ERANGE from the next reader."""
    import torch
    n = 1 << 16
    e = [ctx.generate(f"rmatx:scale=16,ef=16,seed={s}").edges() for s in (1, 2)]
    want = [oracle.cc(n, x) for x in e]
    host = [torch.from_numpy(x.view(np.int32)).pin_memory().numpy().view(np.uint32) for x in e]
    gs = [ctx.graph_from_edges(e[0], n), ctx.graph_from_edges(e[0], n)]
    gs[0].upload_async(host[0])
    for i in range(6):
        if i + 1 < 6:
            gs[(i + 1) % 2].upload_async(host[(i + 1) % 2])
        lab, _ = ctx.cc(gs[i % 2], "baseline-mj")
        assert np.array_equal(lab, want[i % 2]), i
    bad = host[1].copy()
    bad[7, 1] = n
    gs[0].upload_async(bad)
    with pytest.raises(capi.HccError):
        ctx.cc(gs[0], "baseline-mj")
    gs[0].assign(host[0])
    lab, _ = ctx.cc(gs[0], "baseline-mj")
    assert np.array_equal(lab, want[0])
    # three graphs in rotation: the two-entry executable-graph cache misses
    # and re-captures every call, and must still run the right edges
    gs.append(ctx.graph_from_edges(e[1], n))
    for i in range(5):
        lab, _ = ctx.cc(gs[i % 3], "baseline-mj")
        assert np.array_equal(lab, want[[0, 1, 1][i % 3]]), i
    for g in gs:
        g.close()


def test_stale_star_after_a_slot_without_stores(ctx, oracle):
    """Advisor finding (round 1): a middle adaptive slot whose hook stores
    nothing skips its compress, so the star pick must not move the star the
    bitmap tracks.  Slot 0 (m/128 edges) builds a component rooted at 1
    holding half the vertices, slot 1 repeats it (intra-component only:
    no store, no compress), and the rest are (0, x) edges that must pull
    the isolated vertex 0 into that component."""
    n, m = 1 << 16, 1 << 22
    first = m >> 7
    e = np.empty((m, 2), dtype=np.uint32)
    e[:first, 0] = 1
    e[:first, 1] = np.arange(2, first + 2, dtype=np.uint32)
    e[first:5 * first] = np.tile(e[:first], (4, 1))
    rest = m - 5 * first
    e[5 * first:, 0] = 0
    e[5 * first:, 1] = 2 + (np.arange(rest, dtype=np.uint32) % first)
    want = oracle.cc(n, e)
    assert want[1] == 0 and want[first + 1] == 0
    g = ctx.graph_from_edges(e, n)
    import os
    os.environ["HCC_S0B_MIN_LOG2"] = "16"  # the bitmap at this size too
    try:
        lab, mx = ctx.cc(g, "baseline-mj")
    finally:
        os.environ.pop("HCC_S0B_MIN_LOG2", None)
    assert mx["star0_bitmap"]
    assert np.array_equal(lab, want)
    g.close()


def test_graph_cache_survives_buffer_regrowth(ctx, oracle):
    """Advisor finding (round 1): the two cached executable graphs bake the
    worklists, star bitmap and summary into their arguments; a larger graph
    that regrows those buffers must not leave the other cached graph
    pointing at freed memory.  Small n, then larger n (same m), then the
    small one again, several times over."""
    ga = ctx.generate("rmatx:scale=16,ef=64,seed=3")      # n = 2^16, m = 2^22
    gb = ctx.generate("erx:n=2097152,m=4194304,seed=5")   # n = 2^21, m = 2^22
    wa = oracle.cc(ga.n, ga.edges())
    wb = oracle.cc(gb.n, gb.edges())
    import os
    os.environ["HCC_S0B_MIN_LOG2"] = "16"  # both graphs on the bitmap
    try:
        for _ in range(3):
            for g, w in ((ga, wa), (gb, wb)):
                lab, mx = ctx.cc(g, "baseline-mj")
                assert np.array_equal(lab, w)
                assert mx["star0_bitmap"]
    finally:
        os.environ.pop("HCC_S0B_MIN_LOG2", None)
    ga.close()
    gb.close()


@pytest.mark.parametrize("spec", ["rmatx:scale=20,ef=16,seed=7", "erx:n=1100000,m=9000000,seed=3",
                                  "grid:1100x1000", "erx:n=70001,m=40000,seed=9"])
def test_adaptive_streaming_cas_engine(ctx, oracle, spec):
    """The paper's engine on the streaming CAS hook (n >= 2^16): unrolled
    two-launch chains (s <= 64, star pick in the hook's last block, dirty
    flags by segment parity), the device loop (s > 64), the scalar reference
    path (HCC_CAS_STREAM=0) and atomic (s = 1): identical labels."""
    import os
    g = ctx.generate(spec)
    want = oracle.cc(g.n, g.edges())
    for s in (0, 1, 2, 7, 64, 65, 300):
        lab, mx = ctx.cc(g, "adaptive", segments=s)
        assert np.array_equal(lab, want), (spec, s)
        assert mx["components"] == int(np.sum(want == np.arange(g.n, dtype=np.uint32)))
    lab, _ = ctx.cc(g, "atomic")
    assert np.array_equal(lab, want)
    for env in ({"HCC_ADAPT_PICKS": "0"}, {"HCC_ADAPT_PICKS": "64"}, {"HCC_CAS_STREAM": "0"},
                {"HCC_S0B": "0"}):
        os.environ.update(env)
        try:
            lab, _ = ctx.cc(g, "adaptive", segments=9)
            assert np.array_equal(lab, want), (spec, env)
        finally:
            for k in env:
                os.environ.pop(k, None)
    g.close()


@pytest.mark.parametrize("shift", [1, 977])
def test_adaptive_star_moves_off_vertex0(ctx, oracle, shift):
    """Vertex 0 isolated: the adaptive chain's in-hook star pick must move the
    bitmap to the giant's root (or leave it empty) and stay exact."""
    n = 1 << 21
    e = oracle.gen_erx(n - shift, 5, 0, 12 * n).astype(np.uint64) + shift
    g = ctx.graph_from_edges(e.astype(np.uint32), n)
    want = oracle.cc(n, e)
    for s in (0, 4, 31):
        lab, _ = ctx.cc(g, "adaptive", segments=s)
        assert np.array_equal(lab, want), s
    g.close()


@pytest.mark.parametrize("spec", ["rmatx:scale=20,ef=16,seed=7", "erx:n=16777217,m=67108864,seed=2",
                                  "grid:1100x1000", "erx:n=70001,m=40000,seed=9"])
def test_wide_compress_blocks(ctx, oracle, spec):
    """512-thread compress blocks (k_compress_s0b_w, the default from n = 2^26)
    forced on smaller graphs: two 64-word summary chunks per block (shift 0 and,
    at n = 2^24 + 1, shift 1 with shared summary words), partial last block."""
    import os
    g = ctx.generate(spec)
    want = oracle.cc(g.n, g.edges())
    os.environ["HCC_COMP_WIDE"] = "1"
    try:
        for algo in ("baseline-mj", "adaptive"):
            lab, _ = ctx.cc(g, algo)
            assert np.array_equal(lab, want), (spec, algo)
    finally:
        os.environ.pop("HCC_COMP_WIDE", None)
    g.close()


@pytest.mark.parametrize("spec", ["rmatx:scale=20,ef=16,seed=7", "erx:n=16777217,m=67108864,seed=2",
                                  "grid:1100x1000", "erx:n=1048579,m=8000000,seed=5"])
def test_steady_hook_variants(ctx, oracle, spec):
    """The steady slot's hook choices give identical labels: k_hook_sumd by
    sampled summary coverage (default; the worklist passes follow with
    k_hook_cas_sumd), the k_hook_sum / k_hook device vote (HCC_SUM_VOTE=1),
    the plain hook (HCC_SUMD=0), sumd in every streaming slot (HCC_SUMD=2),
    plain worklist passes (HCC_WL_SUMD=0), one-sided walks in the middle
    slots (HCC_HOOK_BOTH=0)."""
    import os
    g = ctx.generate(spec)
    want = oracle.cc(g.n, g.edges())
    for env in ({}, {"HCC_SUM_VOTE": "1"}, {"HCC_SUMD": "0"}, {"HCC_SUMD": "2"},
                {"HCC_SUMD": "1", "HCC_DYN": "0"}, {"HCC_WL_SUMD": "0"}, {"HCC_HOOK_BOTH": "0"}):
        os.environ.update(env)
        try:
            lab, _ = ctx.cc(g, "baseline-mj")
            assert np.array_equal(lab, want), (spec, env)
        finally:
            for k in env:
                os.environ.pop(k, None)
    g.close()
