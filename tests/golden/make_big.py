"""Golden digests for the BASELINE configs too large for a live CPU oracle.

Run here (8 host threads; RMAT-28 takes several minutes):
    python tests/golden/make_big.py [name ...]
For each graph it streams the counter-based generator through the oracle's
streaming DSU (oracle/hookcc_oracle.c oracle_cc_stream, a restatement of
the reference's oracle_cc, proj/include/hookcc/oracle.hpp:17-62; the edge
array is never materialised: RMAT-28 would be 32 GiB packed) and writes
tests/golden/big.json:
    labels_sha256  sha256 of the min-canonical labels as little-endian u32
    components     number of components (vertices with label(v) == v)
    edges_checksum position-keyed checksum of the generated edge stream
                   (oracle_checksum_u32), so the device generator is pinned
                   at full size too
    isolated_root_sample  labels of 64 fixed vertices (a cheap first check)
The oracle itself is pinned against the reference (tests/test_oracle.py);
this file only extends it to sizes the reference cannot hold in this
container's RAM.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle as O  # noqa: E402

SPECS = {
    "rmat28": "rmatx:scale=28,ef=16,seed=1",
    "rmat24": "rmatx:scale=24,ef=16,seed=1",
    "er24": "erx:n=16777216,m=268435456,seed=1",
}


def sample_idx(n: int) -> list[int]:
    rng = np.random.default_rng(28)
    return sorted(int(x) for x in rng.integers(0, n, size=64))


def main(names):
    out_p = HERE / "big.json"
    out = json.loads(out_p.read_text()) if out_p.exists() else {}
    for name in names:
        spec = SPECS[name]
        t = time.time()
        lab, ck, comp = O.cc_stream(spec)
        idx = sample_idx(lab.shape[0])
        out[name] = {
            "spec": spec, "n": int(lab.shape[0]),
            "labels_sha256": hashlib.sha256(lab.astype("<u4").tobytes()).hexdigest(),
            "components": int(comp), "edges_checksum": int(ck),
            "sample_idx": idx, "sample_labels": [int(lab[i]) for i in idx],
            "oracle": "oracle_cc_stream (streaming DSU restatement of oracle.hpp:17-62)",
            "seconds": round(time.time() - t, 1),
        }
        print(name, out[name]["components"], out[name]["seconds"], "s", flush=True)
        out_p.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["rmat24", "er24", "rmat28"])
