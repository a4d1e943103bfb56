#!/usr/bin/env python
"""Summarises an ncu launch list (--metrics gpu__time_duration.sum --csv) of
bench.py: per kernel launches, average time and share of the timed step."""
import collections
import csv
import sys

STEP = ("k_prepare_affine", "k_combine", "k_basis", "k_thickness_pairs", "k_integrals_1d",
        "k_inplane_general", "k_standard", "k_pack_rows")


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    t = collections.defaultdict(list)
    for r in rows:
        name = r[4].split("(")[0]
        t[name].append(float(r[-1]))
    step = {k: sum(v) for k, v in t.items() if any(s in k for s in STEP)}
    tot = sum(step.values())
    print(f"# {cmd}")
    print("# (cold-cache, serialised per-launch times; compare shares, not absolutes).  ncu unit: ns")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot:5.1f}% of step" if k in step else "  outside timed region"
        print(f"{k[:60]:60s} launches={len(v):3d} avg={sum(v) / len(v) / 1e3:10.1f} us {share}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
