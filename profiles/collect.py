#!/usr/bin/env python3
"""Turn one evidence run in gpurun_out/ into the tracked artefacts of profiles/ (run here, after the GPU call):

    python profiles/collect.py r1d          # reads gpurun_out/{bench_TAG.json, bench_TAG_ref.json, launches_TAG.csv, TAG_full_p5/p7.ncu-rep}

writes profiles/TAG_bench_line.json, TAG_bench_reference_arm.json, TAG_launches_p5_p7_p11.csv, TAG_launches_summary.csv,
TAG_ncu_full_p5/p7.txt and profiles/traffic.json (DRAM bytes per hard surface of every kernel, from the ncu --set full capture).
The GPU call that produces the inputs is the one in profiles/README.md.
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1]

shutil.copy(os.path.join(OUT, f"bench_{tag}.json"), os.path.join(HERE, f"{tag}_bench_line.json"))
shutil.copy(os.path.join(OUT, f"bench_{tag}_ref.json"), os.path.join(HERE, f"{tag}_bench_reference_arm.json"))
shutil.copy(os.path.join(OUT, f"launches_{tag}.csv"), os.path.join(HERE, f"{tag}_launches_p5_p7_p11.csv"))
# The reports are reduced on the GPU box (they exceed what gpurun copies back): {tag}_full_pP.{summary.txt, lines.txt, raw.csv}
PRIMES = [p for p in (5, 7, 11) if os.path.exists(os.path.join(OUT, f"{tag}_full_p{p}.raw.csv"))]
for p in PRIMES:
    shutil.copy(os.path.join(OUT, f"{tag}_full_p{p}.summary.txt"), os.path.join(HERE, f"{tag}_ncu_full_p{p}.txt"))
    shutil.copy(os.path.join(OUT, f"{tag}_full_p{p}.lines.txt"), os.path.join(HERE, f"{tag}_ncu_lines_p{p}.txt"))

rows = [r for r in csv.reader(open(os.path.join(OUT, f"launches_{tag}.csv"))) if len(r) > 5]
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None:
        continue
    name, val, unit = r[hdr.index("Kernel Name")], r[hdr.index("Metric Value")].replace(",", ""), r[hdr.index("Metric Unit")]
    try:
        v = float(val)
    except ValueError:
        continue
    ms = v / 1e6 if unit in ("ns", "nsecond") else (v / 1e3 if unit in ("us", "usecond") else v)
    m = re.match(r"(void )?([\w:<>, ()]+?)\(", name)
    a = agg.setdefault(m.group(2) if m else name, [0, 0.0])
    a[0] += 1
    a[1] += ms


def prime(k):
    m = re.search(r"<(\d+)", k)
    return m.group(1) if m else ""


contract = [k for k in agg if not k.startswith("k_free")]
tot = collections.Counter()
for k in contract:
    tot[prime(k)] += agg[k][1]
with open(os.path.join(HERE, f"{tag}_launches_summary.csv"), "w") as fh:
    fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 900, command: python bench.py --steps 2 --warmup 1 --cpu-seconds 1\n")
    fh.write("# (bench.py clamps warm-up to 3: F_5 3 warm-up + 2 timed + e2e calls, then F_7, F_11, then the matrix-free calls; the capture stops at 900 launches).\n")
    fh.write("# Times are cold-cache and serialised by the profiler: compare SHARES per prime with bench.py stage_ms_per_step, not absolutes.\n")
    fh.write("# k_fedder / k_power_full also run in the matrix-free calls, so their share is overstated where k_free appears.\n")
    fh.write("kernel,launches,total_ms,share_of_same_prime\n")
    for k, (n, ms) in agg.items():
        fh.write(f"{k},{n},{ms:.3f},{(ms / tot[prime(k)] if k in contract and tot[prime(k)] else 0):.3f}\n")

def hard_and_batch(p):   # the capture's launch size, from the stats line profiles/run_profile.py prints
    log = open(os.path.join(OUT, f"{tag}_full_p{p}.log")).read()
    return int(re.findall(r"'hard': (\d+)", log)[-1]), int(re.findall(r"'surfaces': (\d+)", log)[-1])


try:
    traffic = json.load(open(os.path.join(HERE, "traffic.json")))
except Exception:
    traffic = {}
for p in PRIMES:
    hard, batch = hard_and_batch(p)
    rows = list(csv.reader(open(os.path.join(OUT, f"{tag}_full_p{p}.raw.csv")).read().splitlines()))
    h, units = rows[0], rows[1]
    traffic[f"p{p}"] = {}
    for r in rows[2:]:
        key = r[h.index("Kernel Name")].split("<")[0].replace("void ", "")

        def val(k):
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "nsecond": 1e-6,
                    "usecond": 1e-3, "msecond": 1}.get(units[h.index(k)], 1)
            return float(r[h.index(k)].replace(",", "")) * mult
        rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
        traffic[f"p{p}"][key] = {"dram_bytes_per_hard_surface": (rd + wr) / hard, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                 "hard_surfaces_in_capture": hard, "gpu_time_ms": t,
                                 "source": f"profiles/{tag}_ncu_full_p{p}.txt (ncu --set full, clock-control none, profiles/run_profile.py --p {p} --batch {batch} --calls 2, second call)"}
json.dump(traffic, open(os.path.join(HERE, "traffic.json"), "w"), indent=1)
d = json.loads(open(os.path.join(HERE, f"{tag}_bench_line.json")).read().strip().splitlines()[-1])
print("F_5", round(d["value"]), {k: round(v, 3) for k, v in d["stage_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"]))
for k, a in d["also"].items():
    if k == "single_surface":
        print(k, {kk: (round(v["ms_per_call"], 3), round(v["cpu_oracle_ms"], 1)) for kk, v in a.items()})
    elif k == "lazy_matrix":
        print(k, {kk: (round(v["value"]), v["built"], v["hard"]) for kk, v in a.items() if kk != "note"})
    elif k != "matrix_free":
        print(k, round(a["value"]), {kk: round(v, 3) for kk, v in a["stage_ms_per_step"].items()}, "frac", round(a["roofline"]["frac"], 3), "e2e", round(a["e2e"]["value"]))
    else:
        print(k, {kk: round(v["value"]) for kk, v in a.items() if kk != "note"})
for p in traffic:
    print(p, {k: (round(v["dram_bytes_per_hard_surface"]), round(v["gpu_time_ms"], 3)) for k, v in traffic[p].items()})
