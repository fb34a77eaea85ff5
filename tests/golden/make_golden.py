"""Generate the committed golden fixtures from the REFERENCE itself.

Run here (where /root/reference exists) after `make -C oracle`:
    python tests/golden/make_golden.py
It drives oracle/_ref/libhookcc_ref.so — the unmodified reference headers
(/root/reference/proj/include/hookcc/*.hpp) compiled by oracle/Makefile —
and writes:
  * fixtures/sample.{el,gr,mtx}: the reference fixture graph
    Graph{6, [(0,1),(1,2),(3,4),(4,5),(0,5)]} (proj/tests/acceptance.cpp:264)
    in the three text formats of io.hpp;
  * golden.json: generator digests, oracle_cc label digests, compute_stats
    and workers=1 engine counters for a set of graphs.
The GPU box has no /root/reference, so tests compare against these files.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle as O  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def write_fixtures():
    fx = HERE / "fixtures"
    fx.mkdir(exist_ok=True)
    edges = [(0, 1), (1, 2), (3, 4), (4, 5), (0, 5)]
    (fx / "sample.el").write_text("# sample graph\n" + "".join(f"{u} {v}\n" for u, v in edges))
    (fx / "sample.gr").write_text("c sample graph\np sp 6 5\n" +
                                  "".join(f"a {u + 1} {v + 1} 1\n" for u, v in edges))
    (fx / "sample.mtx").write_text("%%MatrixMarket matrix coordinate pattern symmetric\n6 6 5\n" +
                                   "".join(f"{u + 1} {v + 1}\n" for u, v in edges))


def graphs():
    """name -> (n, u64 edges) built with the reference generators."""
    rng = np.random.default_rng(20261018)
    out = {
        "rmat16_ef16_s1": (1 << 16, O.ref_gen_rmat(16, 16, 1)),
        "rmat12_ef8_s5": (1 << 12, O.ref_gen_rmat(12, 8, 5)),
        "rmat8_ef8_s23": (1 << 8, O.ref_gen_rmat(8, 8, 23)),
        "grid64x64": (64 * 64, O.ref_gen_grid(64, 64)),
        "grid30x30": (900, O.ref_gen_grid(30, 30)),
        "grid1x7": (7, O.ref_gen_grid(1, 7)),
        "er4096_8192_s7": (4096, O.ref_gen_er(4096, 8192, 7)),
        "er300_600_s17": (300, O.ref_gen_er(300, 600, 17)),
        "er500_3000_s31": (500, O.ref_gen_er(500, 3000, 31)),
    }
    for k in range(6):
        n = int(rng.integers(1, 200))
        m = int(rng.integers(0, 400))
        out[f"rand{k}"] = (n, rng.integers(0, n, size=(m, 2)).astype(np.uint64))
    return out


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: run `make -C oracle` where /root/reference exists")
    write_fixtures()
    gold = {"source": "oracle/_ref/libhookcc_ref.so (unmodified /root/reference headers)",
            "generators": {}, "graphs": {}}
    # generator digests and small literal vectors
    gold["generators"]["rmat_3_2_9"] = O.ref_gen_rmat(3, 2, 9).tolist()
    gold["generators"]["er_4_3_1"] = O.ref_gen_er(4, 3, 1).tolist()
    gold["generators"]["grid_2_2"] = O.ref_gen_grid(2, 2).tolist()
    for name, (n, e) in graphs().items():
        lab = O.ref_cc(n, e)
        bfs = O.ref_bfs_cc(n, e)
        assert np.array_equal(lab, bfs)
        st = O.ref_stats(n, e)
        entry = {"n": n, "m": int(e.shape[0]), "edges_sha256": digest(e),
                 "labels_sha256": digest(lab), "components": int(np.sum(lab == np.arange(n))),
                 "stats": st, "engines": {}}
        if n <= 64:
            entry["edges"] = e.tolist()
            entry["labels"] = lab.tolist()
        if name.startswith("rand"):
            entry["edges"] = e.tolist()
        runs = [("baseline", 0), ("baseline-mj", 0), ("atomic", 0), ("adaptive", 1),
                ("adaptive", 4), ("adaptive", 0)]
        for algo, s in runs:
            if e.shape[0] > 300000 and algo == "baseline":
                continue
            cap = 4096
            l2, mx, segc = O.ref_run(algo, n, e, segments=s, workers=1, seg_cap=cap)
            assert np.array_equal(l2, lab), (name, algo)
            key = algo if algo in ("baseline", "baseline-mj", "atomic") else f"adaptive_s{s}"
            nseg = mx["s"] if algo in ("adaptive", "atomic") else 0
            entry["engines"][key] = {
                "s": mx["s"], "outer_iterations": mx["outer_iterations"],
                "hook_traversal_steps": mx["hook_traversal_steps"],
                "cas_failures": mx["cas_failures"], "jump_steps": mx["jump_steps"],
                "components": mx["components"], "segments_clamped": mx["segments_clamped"],
                "segment_counters": segc[:nseg].tolist() if nseg and nseg <= 64 else None,
            }
        gold["graphs"][name] = entry
        print(name, n, e.shape[0], entry["components"])
    (HERE / "golden.json").write_text(json.dumps(gold, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
