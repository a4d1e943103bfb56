#!/usr/bin/env python
"""Regenerates tests/golden/* from the UNMODIFIED reference compiled here
(oracle/_ref, built from /root/reference by oracle/build_ref.sh).

  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from cases import cases  # noqa: E402
from oracle.checkers import Reference  # noqa: E402
from paper_1905_05417_b200 import problem as P  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Reference()
    arrays = {}
    meta = {}
    for name, (prob, backends) in cases().items():
        for b in backends:
            rp, cols, vals, st = ref.assemble(prob, b, 1, want_stats=True)
            key = f"{name}__{b}"
            arrays[key + "__row_ptr"] = rp
            arrays[key + "__cols"] = cols
            arrays[key + "__values"] = vals
            meta[key] = {"nnz": int(len(vals)), "qpoint_visits": st.qpoint_visits,
                         "frame_evaluations": st.frame_evaluations,
                         "operator_builds": st.operator_builds}
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **arrays)
    # BASELINE C1 / C2: pattern hashes, norms and sampled entries (full CSR is MBs)
    summaries = {}
    rng = np.random.default_rng(20190514)
    for name in ("C1", "C2"):
        prob = P.baseline_config(name)
        for b in (("fast", "standard") if name == "C1" else ("fast",)):
            rp, cols, vals = ref.assemble(prob, b, os.cpu_count() or 1)
            idx = np.sort(rng.choice(len(vals), size=2000, replace=False))
            summaries[f"{name}__{b}"] = {
                "nnz": int(len(vals)), "row_ptr_sha256": digest(rp), "cols_sha256": digest(cols),
                "fro": float(np.sqrt(np.dot(vals, vals))), "max_abs": float(np.abs(vals).max()),
                "sample_idx": idx.tolist(), "sample_values": vals[idx].tolist()}
    # known answers of the reference at the host-setup boundary
    kas = {
        "pagano_D": ref.stiffness(P.pagano(), 0.0).tolist(),
        "baseline_D_45": ref.stiffness(P.baseline_orthotropic(), 0.25 * P.PI).tolist(),
        "bracket_pagano": ref.bracket_parameters(P.pagano()).tolist(),
        "angle_decomposition_pagano": ref.angle_decomposition(P.pagano()).tolist(),
        "contraction_table_pagano_0.6": ref.contraction_table(P.pagano(), 0.6).tolist(),
    }
    with open(os.path.join(HERE, "ref_summaries.json"), "w") as f:
        json.dump({"small": meta, "baseline": summaries, "known_answers": kas}, f, indent=1)
    print("wrote", os.path.join(HERE, "ref_small.npz"), "and ref_summaries.json")


if __name__ == "__main__":
    main()
