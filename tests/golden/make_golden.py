"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref, the unmodified
/root/reference/proj/core sources compiled in place). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed, small):
  products.npz  -- A, B inputs from spgemm::random_csr (libstdc++ mt19937_64 distributions),
                   C = spgemm::multiply(A, B) and its stats (total_nprod, nnz, spilled_rows)
  binning.npz   -- spgemm::run_binning on random metrics for every preset (deterministic mode)
  kat.json      -- known answers: presets, spill constructions, hand cases (test_pipeline.cpp)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402

# (rows_a, cols_a=rows_b, cols_b, density_a, density_b, seed) -- shapes of test_pipeline.cpp:170-184,
# acceptance criterion 2 (acceptance_main.cpp:142-197) and rectangular cases
CASES = [
    (120, 120, 120, 0.05, 0.05, 33),
    (257, 140, 301, 0.05, 0.04, 34),
    (400, 400, 400, 0.03, 0.03, 35),
    (31, 400, 77, 0.08, 0.05, 36),
    (600, 600, 600, 0.015, 0.015, 0xACCE507),
    (509, 509, 509, 0.0099, 0.0099, 0xACCE508),
    (1, 50, 50, 0.5, 0.3, 37),
    (300, 1, 300, 1.0, 0.02, 38),
]


def main():
    if not O.ref_available():
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    arrays = {}
    meta = []
    for idx, (m, k, n, da, db, seed) in enumerate(CASES):
        a = O.ref_random_csr(m, k, da, seed)
        b = O.ref_random_csr(k, n, db, seed + 1000)
        c, info = O.ref_multiply(a, b)
        for tag, mat in (("a", a), ("b", b), ("c", c)):
            arrays[f"{idx}_{tag}_rpt"] = mat.rpt
            arrays[f"{idx}_{tag}_col"] = mat.col
            arrays[f"{idx}_{tag}_val"] = mat.val
            arrays[f"{idx}_{tag}_shape"] = np.array([mat.rows, mat.cols], np.int64)
        nprod = O.ref_rpt_region(a, b, 1)
        arrays[f"{idx}_nprod"] = nprod
        meta.append(dict(total_nprod=info["total_nprod"], nnz=info["nnz_of_product"],
                         spilled_rows=info["spilled_rows"], cr=info["cr"]))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "products.npz"), **arrays)

    rng = np.random.default_rng(13)
    bins = {}
    presets = [(0, "sym_1x"), (0, "sym_1.2x"), (0, "sym_1.5x"), (1, "num_1x"), (1, "num_1.5x"),
               (1, "num_2x"), (1, "num_3x")]
    for phase, name in presets:
        for trial, hi in enumerate((15, 40000)):
            metric = rng.integers(0, hi + 1, 1 + int(rng.integers(0, 3000))).astype(np.int64)
            r = O.ref_run_binning(metric, phase, name, True, 128)
            key = f"{name}_{trial}"
            bins[key + "_metric"] = metric
            bins[key + "_bins"] = r["bins"]
            bins[key + "_info"] = np.concatenate([r["bin_size"], r["bin_offset"],
                                                  [r["max_metric"], r["total_metric"], int(r["fast_path"])]])
    np.savez_compressed(os.path.join(HERE, "binning.npz"), **bins)

    kat = {"presets": {}}
    for phase, name in presets:
        up, tab = O.preset(phase, name)  # pinned below against the reference's own preset()
        kat["presets"][name] = {"upper": [int(x) for x in up], "table_size": [int(x) for x in tab]}
    # spill constructions of test_pipeline.cpp:29-43 (built in numpy by the tests)
    from helpers import spill_pair  # noqa: E402
    kat["spill"] = {}
    for distinct, rows_in_b in ((20000, 200), (19660, 20), (6000, 60)):
        a, b = spill_pair(distinct, rows_in_b)
        c, info = O.ref_multiply(a, b, workers=2)
        kat["spill"][f"{distinct}_{rows_in_b}"] = dict(spilled_rows=info["spilled_rows"],
                                                       row0_nnz=int(c.rpt[1] - c.rpt[0]),
                                                       nnz=info["nnz_of_product"],
                                                       total_nprod=info["total_nprod"])
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
