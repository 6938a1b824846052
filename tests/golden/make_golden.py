"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libdmm_ref.so (the reference headers compiled in place by
oracle/Makefile) and records inputs, outputs and reports of the reference's own
public API (gen_instance, run_algorithm, integer_sort_general, permute, layout
primitives) into tests/golden/golden.npz.  The fixtures are small and committed;
the GPU box never needs /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import PARTITION_GENERAL, PERMUTE, Port, Ref  # noqa: E402

PARTITION_CASES = [(32, 32, s) for s in range(4)] + [(32, 16, s) for s in range(4)] + [
    (32, 64, 0), (16, 16, 0), (64, 16, 0), (64, 64, 0), (2, 4, 0), (3, 9, 0), (8, 8, 0), (256, 16, 0)]
# (w, m, seed, domain) -- permute-kind instances sorted as integer keys, and uint32 tiles
INTSORT_CASES = [(32, 16, 0, 512), (32, 32, 1, 1024), (64, 16, 2, 1024)]
U32SORT_CASES = [(32, 128, 0), (32, 128, 1), (32, 32, 2)]
PERMUTE_CASES = [(32, 32, s) for s in range(1, 7)] + [(32, 16, s) for s in range(1, 7)] + [
    (32, 2, 1), (32, 4, 1), (64, 16, 1), (64, 8, 1), (128, 64, 1)]
# PartitionProbe snapshots (after_balance / after_divide of the outer recursion):
# (w, m, seed, domain); domain = w on partition instances is partition_general's recursion
PROBE_CASES = [(32, 16, 0, 32), (32, 16, 1, 32), (32, 16, 2, 32), (16, 8, 0, 16), (16, 8, 3, 16),
               (32, 16, 4, 512)]
LAYOUT_CASES = [("to_column_major", 2, 4), ("to_row_major", 2, 4), ("to_column_major", 32, 8),
                ("to_row_major", 8, 32), ("transpose_square", 32, 32), ("to_column_major", 3, 6)]


def main() -> None:
    ref = Ref()
    port = Port()
    arrays: dict[str, np.ndarray] = {}
    meta: dict[str, object] = {"partition": [], "intsort": [], "u32sort": [], "permute": [], "layout": [],
                               "probe": []}

    for (w, m, s) in PARTITION_CASES:
        g = ref.gen_instance(1, w, m, s)
        st, out, rep = ref.partition_general(g)
        key = f"partition_{w}x{m}_s{s}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        _, _, run = ref.run_algorithm(PARTITION_GENERAL, g, s)
        meta["partition"].append({"key": key, "w": w, "m": m, "seed": s, "status": st, **rep,
                                  "steps": run["steps"], "correct": run["correct"]})

    for (w, m, s, dom) in INTSORT_CASES:
        g = ref.gen_instance(2, w, m, s)
        st, out, rep = ref.integer_sort_general(g, dom)
        key = f"intsort_{w}x{m}_s{s}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        meta["intsort"].append({"key": key, "w": w, "m": m, "seed": s, "domain": dom, "status": st, **rep})

    for (w, m, s) in U32SORT_CASES:
        g = port.gen_sort_u32(w, m, s)  # builder-defined uint32 generator
        st, out, rep = ref.integer_sort_general(g, 1 << 32)
        key = f"u32sort_{w}x{m}_s{s}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        meta["u32sort"].append({"key": key, "w": w, "m": m, "seed": s, "status": st, **rep})

    for (w, m, s) in PERMUTE_CASES:
        g = ref.gen_instance(2, w, m, s)
        st, out, rep = ref.run_algorithm(PERMUTE, g, s)
        key = f"permute_{w}x{m}_s{s}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        pipe = rep["pipeline"]
        meta["permute"].append({"key": key, "w": w, "m": m, "seed": s, "status": st, "steps": rep["steps"],
                                "correct": rep["correct"], **pipe})

    for (w, m, s, dom) in PROBE_CASES:
        g = ref.gen_instance(1 if dom == w else 2, w, m, s)
        st, out, rep = ref.integer_sort_general(g, dom, probe_snaps=16)
        key = f"probe_{w}x{m}_s{s}_d{dom}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        arrays[key + "_snaps"] = rep["snapshots"].astype(np.uint32)
        meta["probe"].append({"key": key, "w": w, "m": m, "seed": s, "domain": dom, "status": st,
                              "cleanup_retries": rep["cleanup_retries"], "n_snaps": int(rep["snapshots"].shape[0])})

    for (op, w, m) in LAYOUT_CASES:
        g = np.arange(1, w * m + 1, dtype=np.uint64).reshape(w, m)
        st, out = ref.layout(op, g)
        key = f"layout_{op}_{w}x{m}"
        arrays[key + "_in"] = g.astype(np.uint32)
        arrays[key + "_out"] = out.astype(np.uint32)
        meta["layout"].append({"key": key, "op": op, "w": w, "m": m, "status": st})

    meta["mt19937_64"] = {str(seed): [str(x) for x in port.mt19937_64(seed, 16)] for seed in (1, 5489, 777)}
    meta["mt19937_64_10000th_default"] = str(port.mt19937_64(5489, 10000)[-1])
    meta["shape_ok"] = {f"{W}x{M}": ref.general_sort_shape_ok(W, M) for (W, M) in
                        [(32, 8), (32, 16), (32, 32), (256, 32), (32, 4), (4096, 16), (2048, 8)]}
    meta["permute_threshold"] = {f"{w}x{m}": ref.permute_threshold(w, m) for (w, m) in
                                 [(32, 32), (32, 16), (128, 64), (4096, 64)]}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, meta keys {sorted(meta)}")


if __name__ == "__main__":
    main()
