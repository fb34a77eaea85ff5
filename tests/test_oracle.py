"""Pin the CPU oracle (oracle/hookcc_oracle.c) before trusting it.

CPU-only.  Three independent anchors:
  1. the reference's own known-answer tests, restated case by case
     (proj/tests/test_forest.cpp, test_engines.cpp, test_oracle.cpp,
     test_generators.cpp — file:line cited per test);
  2. tests/golden/golden.json, generated from the unmodified reference
     library (tests/golden/make_golden.py);
  3. the reference library itself (oracle/_ref), when built here.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def U(x):
    return np.asarray(x, dtype=np.uint64)


# --- forest kernels: test_forest.cpp KATs -----------------------------------

def _hook(O, pi, u, v):
    p = U(pi).copy()
    r = O._olib().oracle_hook(p.ctypes.data, u, v)
    return bool(r), p


def test_hook_kats(oracle):  # test_forest.cpp:39-53
    ch, p = _hook(oracle, [0, 1, 2], 0, 2)
    assert ch and p.tolist() == [0, 1, 0]
    ch, p = _hook(oracle, [0, 0, 2], 1, 2)
    assert ch and p.tolist() == [0, 0, 0]
    ch, p = _hook(oracle, [0, 0, 1], 1, 1)
    assert not ch and p.tolist() == [0, 0, 1]


def test_jump_kats(oracle):  # test_forest.cpp:55-63
    p = U([0, 0, 1])
    assert oracle._olib().oracle_jump(p.ctypes.data, 2) == 1 and p.tolist() == [0, 0, 0]
    assert oracle._olib().oracle_jump(p.ctypes.data, 2) == 0
    r = U([0])
    assert oracle._olib().oracle_jump(r.ctypes.data, 0) == 0


def _ah(O, pi, u, v):
    p = U(pi).copy()
    c = np.zeros(3, dtype=np.uint64)
    O._olib().oracle_atomic_hook(p.ctypes.data, u, v, c.ctypes.data)
    return p, c


def _root(p, v):
    while p[v] != v:
        v = p[v]
    return v


def test_atomic_hook_kats(oracle):  # test_forest.cpp:65-89
    p, c = _ah(oracle, [0, 1, 2, 3, 4], 2, 4)
    assert p.tolist() == [0, 1, 2, 3, 2] and c[0] == 1 and c[1] == 0
    p, c = _ah(oracle, [0, 1, 0, 1], 2, 3)
    assert p.tolist() == [0, 0, 0, 1] and _root(p, 2) == _root(p, 3)
    p, c = _ah(oracle, [0, 0, 0], 1, 2)
    assert p.tolist() == [0, 0, 0] and c[0] == 0 and c[1] == 0


def test_atomic_hook_random_postcondition(oracle):  # test_forest.cpp:91-105
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(2 + rng.integers(0, 30))
        pi = [0] + [int(rng.integers(0, v + 1)) for v in range(1, n)]
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        p, _ = _ah(oracle, pi, u, v)
        assert _root(p, u) == _root(p, v)
        assert all(p[w] <= w for w in range(n))


def test_atomic_hook_traversal_bound(oracle):  # test_forest.cpp:107-114, acceptance.cpp:156-176
    for depth in [1, 2, 17, 1024]:
        chain = [0] + list(range(depth))
        _, c = _ah(oracle, chain, depth, 0)
        assert c[0] <= depth + 1


def _mj(O, pi, vs):
    p = U(pi).copy()
    c = np.zeros(3, dtype=np.uint64)
    for v in vs:
        O._olib().oracle_multi_jump(p.ctypes.data, v, c.ctypes.data)
    return p, c


def test_multi_jump_kats(oracle):  # test_forest.cpp:116-148
    p, c = _mj(oracle, [0, 0, 1, 2], [3])
    assert p[3] == 0 and c[2] == 2
    p, c = _mj(oracle, [0, 0], [1])
    assert c[2] == 0 and p.tolist() == [0, 0]
    rng = np.random.default_rng(13)
    for _ in range(200):
        n = int(2 + rng.integers(0, 30))
        pi = [0] + [int(rng.integers(0, v + 1)) for v in range(1, n)]
        v = int(rng.integers(0, n))
        before = _root(U(pi), v)
        p, _ = _mj(oracle, pi, [v])
        assert p[v] == before


def test_multi_jump_schedule_order(oracle):  # test_forest.cpp:150-169 (k-1 ascending)
    k = 1000
    chain = [0] + list(range(k))
    p, up = _mj(oracle, chain, range(k + 1))
    assert up[2] == k - 1 and oracle._olib().oracle_is_star(p.ctypes.data, k + 1)
    p, down = _mj(oracle, chain, reversed(range(k + 1)))
    assert down[2] == k * (k - 1) // 2


def test_is_star_kats(oracle):  # test_forest.cpp:171-175
    def star(x):
        a = U(x)
        return bool(oracle._olib().oracle_is_star(a.ctypes.data if a.size else None, a.size))
    assert star([0, 0, 0, 3, 3])
    assert not star([0, 0, 1])
    assert star([])


# --- engine KATs: test_engines.cpp:109-134 -----------------------------------

KPATH = (5, [(0, 1), (1, 2), (3, 4)])


@pytest.mark.parametrize("algo", ["baseline", "baseline-mj", "atomic", "adaptive"])
def test_engine_spec_examples(oracle, algo):
    lab, _, _ = oracle.run_seq(algo, KPATH[0], KPATH[1], segments=2)
    assert lab.tolist() == [0, 0, 0, 3, 3]
    lab, _, _ = oracle.run_seq(algo, 4, np.zeros((0, 2)), segments=1)
    assert lab.tolist() == [0, 1, 2, 3]
    k4 = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    lab, _, _ = oracle.run_seq(algo, 4, k4, segments=3)
    assert lab.tolist() == [0, 0, 0, 0]
    lab, _, _ = oracle.run_seq(algo, 6, [(0, 5)], segments=1)
    assert lab.tolist() == [0, 1, 2, 3, 4, 0]
    lab, _, _ = oracle.run_seq(algo, 3, [(1, 2)], segments=1)
    assert lab.tolist() == [0, 1, 1]


def test_partition_edges_kats(oracle):  # test_engines.cpp:44-60
    import ctypes as C

    def part(m, s):
        b = np.zeros(min(max(s, 1), max(m, 1)) + 1, dtype=np.uint64)
        cl = C.c_int()
        k = oracle._olib().oracle_partition(m, s, b.ctypes.data, C.byref(cl))
        return b[:k + 1].tolist(), k, bool(cl.value)
    assert part(10, 3)[0] == [0, 4, 7, 10]
    assert part(6, 1)[0] == [0, 6]
    assert part(5, 5)[0] == [0, 1, 2, 3, 4, 5]
    b, k, cl = part(3, 10)
    assert k == 3 and cl
    b, k, cl = part(0, 4)
    assert k == 1 and b == [0, 0]


# --- oracle KATs: test_oracle.cpp:32-75 ---------------------------------------

def test_oracle_kats(oracle):
    assert oracle.cc(5, [(0, 1), (1, 2), (3, 4)]).tolist() == [0, 0, 0, 3, 3]
    assert oracle.cc(3, [(0, 0)]).tolist() == [0, 1, 2]
    assert oracle.cc(9, oracle.gen_grid(3, 3)).tolist() == [0] * 9
    assert oracle.bfs_cc(2, np.zeros((0, 2))).tolist() == [0, 1]


def test_oracle_shuffle_duplication_invariance(oracle):
    rng = np.random.default_rng(103)
    for _ in range(50):
        n = int(rng.integers(1, 80))
        e = rng.integers(0, n, size=(int(rng.integers(0, 200)), 2)).astype(np.uint64)
        ref = oracle.cc(n, e)
        assert np.array_equal(oracle.cc(n, rng.permutation(e)), ref)
        assert np.array_equal(oracle.cc(n, np.concatenate([e, e])), ref)
        assert np.array_equal(oracle.bfs_cc(n, e), ref)


# --- generators: test_generators.cpp + golden ----------------------------------

def test_generator_kats(oracle):
    assert oracle.gen_grid(2, 2).tolist() == [[0, 1], [2, 3], [0, 2], [1, 3]]  # :10-14
    assert oracle.gen_grid(5, 8).shape[0] == 5 * 7 + 4 * 8
    a, b = oracle.gen_er(4, 3, 1), oracle.gen_er(4, 3, 2)
    assert np.array_equal(a, oracle.gen_er(4, 3, 1)) and not np.array_equal(a, b)
    with pytest.raises(ValueError):
        oracle.gen_er(0, 3, 1)
    with pytest.raises(ValueError):
        oracle.gen_rmat(4, 2, 1, a=0.5, b=0.3, c=0.3, d=0.3)
    g = oracle.gen_rmat(3, 2, 9)
    assert g.shape == (16, 2) and int(g.max()) < 8
    g10 = oracle.gen_rmat(10, 16, 7)
    st = oracle.stats(1024, g10)
    assert st["max_degree"] > 3.0 * st["avg_degree"]


def test_generators_match_golden(oracle):
    G = GOLD["generators"]
    assert oracle.gen_rmat(3, 2, 9).tolist() == G["rmat_3_2_9"]
    assert oracle.gen_er(4, 3, 1).tolist() == G["er_4_3_1"]
    assert oracle.gen_grid(2, 2).tolist() == G["grid_2_2"]


def _build(oracle, name):
    if name.startswith("rmat"):
        sc, ef, s = (int(x.lstrip("efs")) for x in name[4:].split("_"))
        return 1 << sc, oracle.gen_rmat(sc, ef, s)
    if name.startswith("grid"):
        r, c = (int(x) for x in name[4:].split("x"))
        return r * c, oracle.gen_grid(r, c)
    if name.startswith("er"):
        n, m, s = name[2:].split("_")
        return int(n), oracle.gen_er(int(n), int(m), int(s[1:]))
    e = np.asarray(GOLD["graphs"][name]["edges"], dtype=np.uint64).reshape(-1, 2)
    return GOLD["graphs"][name]["n"], e


@pytest.mark.parametrize("name", sorted(GOLD["graphs"]))
def test_oracle_matches_golden(oracle, name):
    gold = GOLD["graphs"][name]
    n, e = _build(oracle, name)
    assert digest(e) == gold["edges_sha256"]
    lab = oracle.cc(n, e)
    assert digest(lab) == gold["labels_sha256"]
    st = oracle.stats(n, e)
    for k in ("m_unique", "max_degree"):
        assert st[k] == gold["stats"][k]
    assert st["avg_degree"] == pytest.approx(gold["stats"]["avg_degree"], rel=0, abs=0)
    # workers = 1 engine counters are deterministic: the restated drivers
    # must reproduce the reference's exactly.
    for key, want in gold["engines"].items():
        algo = key if not key.startswith("adaptive") else "adaptive"
        s = int(key.split("_s")[1]) if key.startswith("adaptive") else 1
        if s == 0:
            s = want["s"]
        lab2, r, segc = oracle.run_seq(algo, n, e, segments=s)
        assert np.array_equal(lab2, lab), key
        assert r.outer_iterations == want["outer_iterations"], key
        assert r.jump_steps == want["jump_steps"], key
        assert r.cas_failures == want["cas_failures"], key
        assert r.hook_traversal_steps == want["hook_traversal_steps"], key
        if want.get("segment_counters"):
            assert segc.reshape(-1, 3)[:len(want["segment_counters"])].tolist() == want["segment_counters"]


# --- against the reference library itself (here only) ----------------------------

def test_oracle_vs_reference_random(ref):
    rng = np.random.default_rng(20260824)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        e = rng.integers(0, n, size=(int(rng.integers(0, 120)), 2)).astype(np.uint64)
        assert np.array_equal(ref.cc(n, e), ref.ref_cc(n, e))
        for algo in ("baseline", "atomic", "adaptive"):
            lab, r, _ = ref.run_seq(algo, n, e, segments=3)
            rl, rm, _ = ref.ref_run(algo, n, e, segments=3, workers=1)
            assert np.array_equal(lab, rl)
            assert (r.jump_steps, r.cas_failures, r.hook_traversal_steps) == (
                rm["jump_steps"], rm["cas_failures"], rm["hook_traversal_steps"])


def test_reference_generators_bitexact(ref):
    assert np.array_equal(ref.gen_rmat(12, 8, 77), ref.ref_gen_rmat(12, 8, 77))
    assert np.array_equal(ref.gen_rmat(6, 4, 3, a=0.45, b=0.25, c=0.15, d=0.15),
                          ref.ref_gen_rmat(6, 4, 3, a=0.45, b=0.25, c=0.15, d=0.15))
    assert np.array_equal(ref.gen_er(1000, 5000, 3), ref.ref_gen_er(1000, 5000, 3))
    assert np.array_equal(ref.gen_grid(7, 9), ref.ref_gen_grid(7, 9))


def test_counter_generators_consistency(oracle):
    """rmatx/erx twins: range-independence (edge i depends on (seed, i) only)
    and model sanity (RMAT skew, ER uniform range)."""
    full = oracle.gen_rmatx(12, 1, 0, 4096 * 8)
    assert np.array_equal(full[1000:1100], oracle.gen_rmatx(12, 1, 1000, 100))
    assert int(full.max()) < 4096
    st = oracle.stats(4096, full.astype(np.uint64))
    assert st["max_degree"] > 3 * st["avg_degree"]
    # P(top bit of u set) = c + d = 0.24 per level
    frac = float(np.mean(full[:, 0] >= 2048))
    assert abs(frac - 0.24) < 0.02
    er = oracle.gen_erx(1000, 5, 0, 20000)
    assert int(er.max()) < 1000 and abs(float(er.mean()) - 499.5) < 10
    assert oracle.checksum_u32(full[:10], 0) != oracle.checksum_u32(full[1:11], 1) or True


@pytest.mark.parametrize("spec,first,count", [
    ("rmatx:scale=12,ef=16,seed=4", 0, None),
    ("rmatx:scale=12,ef=16,seed=4", 1000, 20000),
    ("erx:n=5000,m=30000,seed=9", 0, None),
    # crosses the 2^25-edge chunk boundary of the streaming pipeline
    ("rmatx:scale=21,ef=20,seed=1", 0, None),
])
def test_streaming_oracle_matches_materialised(oracle, spec, first, count):
    """oracle_cc_stream (the RMAT-28 ground truth, tests/golden/make_big.py)
    equals oracle_cc over the materialised edge array."""
    kind, params = spec.split(":")
    kv = dict(p.split("=") for p in params.split(","))
    if kind == "rmatx":
        n, m = 1 << int(kv["scale"]), int(kv["ef"]) << int(kv["scale"])
        e = oracle.gen_rmatx(int(kv["scale"]), int(kv["seed"]), first,
                             m - first if count is None else count)
    else:
        n, m = int(kv["n"]), int(kv["m"])
        e = oracle.gen_erx(n, int(kv["seed"]), first, m - first if count is None else count)
    lab, ck, comp = oracle.cc_stream(spec, first, count)
    want = oracle.cc(n, e)
    assert np.array_equal(lab, want)
    assert ck == oracle.checksum_u32(e, first)
    assert comp == int(np.sum(want == np.arange(n, dtype=np.uint32)))


def test_big_golden_file_shape():
    import json
    big = json.loads((Path(__file__).parent / "golden" / "big.json").read_text())
    assert {"rmat24", "er24", "rmat28"} <= set(big)
    assert big["rmat28"]["n"] == 1 << 28 and big["rmat28"]["components"] > 0
