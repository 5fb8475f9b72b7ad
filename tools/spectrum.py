#!/usr/bin/env python3
"""Height-spectrum search (BASELINE.json configs[3]; paper section 7): sample seeded random quartics over F_p
until every height 1..10 and infinity has been seen, print one witness per height in the fixture-table format.

    python tools/spectrum.py --p 7 --block 1000000 --max-blocks 400 [--devices 0,1,...] [--method naive] [--out FILE]

The witnesses it writes (fixture-table rows) are re-verified by the CPU oracle in the test suite
(tests/test_oracle_golden.py::test_spectrum_witnesses); this tool itself never touches oracle/.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_12428_b200 as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=5)
    ap.add_argument("--block", type=int, default=1000000)
    ap.add_argument("--max-blocks", type=int, default=100)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--devices", default="0")
    ap.add_argument("--method", choices=("matrix", "naive", "lazy"), default="matrix",
                    help="matrix: operator matrix in HBM + matvec chain (contract path); naive: matrix-free iteration")
    ap.add_argument("--want", default=None, help="comma-separated heights to look for (inf allowed); default 1..10,inf")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    devs = [int(x) for x in a.devices.split(",")]
    t0 = time.perf_counter()

    def progress(n, hist, wit):
        if n % 10 == 0:
            print(f"[{time.perf_counter() - t0:7.1f}s] blocks {n} samples {hist.total} seen {sorted(wit)}", file=sys.stderr, flush=True)

    want = None if a.want is None else [float("inf") if t == "inf" else int(t) for t in a.want.split(",")]
    wit, hist, blocks = q.spectrum_search(a.p, a.block, a.seed, 10, a.max_blocks, devices=devs, progress=progress,
                                          method=a.method, want=want)
    dt = time.perf_counter() - t0
    rows = q.spectrum_rows(wit)
    print(rows)
    summary = {"p": a.p, "method": a.method, "seed": a.seed, "block": a.block, "blocks": blocks, "samples": hist.total, "seconds": dt,
               "surfaces_per_s": hist.total / dt, "histogram": hist.as_dict(), "complete": (set(range(11)) if want is None else {0 if h == float("inf") else h for h in want}) <= set(wit),
               "witnesses": {("inf" if h == 0 else str(h)): {"block": b, "index": i} for h, (b, i, _) in sorted(wit.items())}}
    print(json.dumps(summary), file=sys.stderr)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(rows + "\n")
            fh.write("# " + json.dumps(summary) + "\n")


if __name__ == "__main__":
    main()
