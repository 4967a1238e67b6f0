"""Writes the remask-selection parity record for BASELINE configs[0-2]
(tests/selection_cases.py): {config, layout, M, k, band_rows, mismatches, ...}
per case, every masked row against the fp64 CPU oracle.

    python scripts/selection_parity.py --out profiles/r02_selection_parity.json
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]

import torch  # noqa: E402

import selection_cases as sc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--cases", default="tiny,llada_32k:scattered,llada_32k:suffix,dream_128k:scattered,"
                                       "dream_128k:suffix")
    args = ap.parse_args()
    from paper_2601_06562_b200 import _build

    _build.build()
    dev = torch.device("cuda", 0)
    recs = []
    for case in args.cases.split(","):
        rec = sc.tiny_case(dev) if case == "tiny" else sc.head_case(dev, *case.split(":"))
        try:
            sc.check(rec)
            rec["passes_bar"] = True
        except AssertionError:
            rec["passes_bar"] = False
        print(json.dumps(rec), flush=True)
        recs.append(rec)
    out = {"host_cores": len(os.sched_getaffinity(0)), "band_rel": sc.BAND_REL, "cases": recs}
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
