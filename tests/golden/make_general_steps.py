"""Golden fixtures for the recursion's step meter (dmm_general_steps), from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_general_steps.py
Records, per case, the input grid, the domain, Machine::steps(), GeneralStats::cleanup_retries
and the final grid of the reference's integer_sort_general (partition.hpp:436; partition_general
is the same call with domain = w) into tests/golden/general_steps.npz:
  * partition instances (gen_instance kind partition, run_algorithm's partition_general) and
    permute-kind instances sorted as integer keys (run_algorithm's integer_sort_general,
    domain w m) on the recursion shapes w > m;
  * random keys on small-m shapes where the checked cleanup retries (cleanup_retries > 0).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import ALGORITHMS, Ref  # noqa: E402

SHAPES = [(32, 16), (64, 16), (16, 8), (64, 8), (64, 32), (128, 32), (256, 16), (128, 64)]
RETRY_SHAPES = [(8, 2), (16, 2), (16, 4), (32, 4), (64, 4)]


def main() -> None:
    ref = Ref()
    rng = np.random.default_rng(20261019)
    cases: dict[str, list] = {}

    def add(w, m, grid, domain, steps, retries, out):
        c = cases.setdefault(f"{w}x{m}", [])
        c.append((grid.astype(np.uint32), domain, steps, retries, out.astype(np.uint32)))

    for (w, m) in SHAPES:
        n = 8 if w * m >= 4096 else 16
        for seed in range(n):
            g = ref.gen_instance(1, w, m, seed)
            s, out, rep = ref.run_algorithm(ALGORITHMS["partition_general"], g, seed)
            assert s == 0 and rep["correct"], (w, m, seed, s)
            s2, out2, r2 = ref.integer_sort_general_steps(g, w, enforce_pre=True, strict=True)
            assert s2 == 0 and r2["steps"] == rep["steps"]
            add(w, m, g, w, rep["steps"], rep["cleanup_retries"], out2)
        for seed in range(4):
            g = ref.gen_instance(2, w, m, seed)
            s, out, rep = ref.run_algorithm(ALGORITHMS["integer_sort_general"], g, seed)
            assert s == 0 and rep["correct"], (w, m, seed, s)
            s2, out2, r2 = ref.integer_sort_general_steps(g, w * m, enforce_pre=True, strict=True)
            assert s2 == 0 and r2["steps"] == rep["steps"]
            add(w, m, g, w * m, rep["steps"], rep["cleanup_retries"], out2)
    for (w, m) in RETRY_SHAPES:
        got = 0
        for t in range(400):
            domain = int(rng.choice([2, w, w * m, 1 << 20]))
            g = rng.integers(0, domain, size=(w, m))
            s, out, rep = ref.integer_sort_general_steps(g, domain)
            if s != 0 or (rep["cleanup_retries"] == 0 and t % 4):
                continue
            add(w, m, g, domain, rep["steps"], rep["cleanup_retries"], out)
            got += 1
            if got == 24:
                break

    arrays = {}
    for key, cs in cases.items():
        arrays[key + "_in"] = np.stack([c[0] for c in cs])
        arrays[key + "_domain"] = np.array([c[1] for c in cs], dtype=np.uint64)
        arrays[key + "_steps"] = np.array([c[2] for c in cs], dtype=np.uint64)
        arrays[key + "_retries"] = np.array([c[3] for c in cs], dtype=np.uint32)
        arrays[key + "_out"] = np.stack([c[4] for c in cs])
    np.savez_compressed(os.path.join(HERE, "general_steps.npz"), **arrays)
    for key, cs in cases.items():
        print(key, len(cs), "cases; retries > 0:", sum(c[3] > 0 for c in cs),
              "; distinct steps:", len({c[2] for c in cs}))


if __name__ == "__main__":
    main()
