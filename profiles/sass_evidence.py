#!/usr/bin/env python3
"""SASS evidence for the hot kernels of libqfs.so, produced without a GPU (cuobjdump -sass on the shipped library):

    python profiles/sass_evidence.py [tag]        # writes profiles/<tag>_sass.txt   (default tag: r2)

Per kernel: instruction count, opcode histogram, and every instruction of the classes that prove the Blackwell-side claims of
DESIGN.md -- IMMA (int8 tensor-core MMA of the Witt carry), UBLKCP (cp.async.bulk: TMA-engine bulk copies), SYNCS (mbarrier),
IDP (DP4A), REDUX -- with its address, plus the inner loop of the Witt-carry tile (between the first and last IMMA of a tile).
"""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(HERE), "paper_2502_12428_b200", "libqfs.so")
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
HOT = ["k_delta_mma", "k_matrix_staged", "k_chain", "k_chain_grid", "k_power_full", "k_fedder", "k_delta_box", "k_delta_prep",
       "k_sample_quartics", "k_free"]
MARK = ("IMMA", "UBLKCP", "UBLKPF", "SYNCS", "IDP", "REDUX", "UTMA", "UTC", "LDSM", "HMMA")

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if cur and m:
        funcs[cur].append((m.group(1), m.group(2).strip()))
demangled = subprocess.run(["cu++filt"] + list(funcs), capture_output=True, text=True).stdout.splitlines()
names = dict(zip(funcs, demangled)) if len(demangled) == len(funcs) else {f: f for f in funcs}

out = [f"# cuobjdump -sass {os.path.relpath(LIB, os.path.dirname(HERE))}   (nvcc -gencode arch=compute_100a,code=sm_100a; python profiles/sass_evidence.py {tag})", ""]
for f, ins in funcs.items():
    name = names[f]
    m = re.match(r"^(?:void )?([\w:]+)(<[^>]*>)?", name)
    if not m:
        continue
    base, targs = m.group(1), (m.group(2) or "").replace("(int)", "").replace("(bool)", "")
    short = base + targs
    if base not in HOT or (targs and not re.match(r"<(5|7|11)\b", targs)):
        continue
    ops = collections.Counter(re.sub(r"^@!?U?P\d+\s+", "", i[1]).split()[0].split(".")[0] for i in ins)
    out.append(f"== {short}: {len(ins)} instructions")
    out.append("   opcodes: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(24)))
    marks = [(a, t) for a, t in ins if any(k in t.split()[0] or (t.startswith("@") and k in t) for k in MARK)]
    by = collections.Counter(re.sub(r"^@!?U?P\d+\s+", "", t).split()[0] for _, t in marks)
    out.append("   marked:  " + (", ".join(f"{k} x{v}" for k, v in by.most_common()) or "none"))
    for a, t in marks[:6]:
        out.append(f"      /*{a}*/ {t}")
    if short == "k_delta_mma<5>":
        idx = [i for i, (_, t) in enumerate(ins) if "IMMA" in t]
        # the last unrolled tile body: from its four LDS.64 of the B fragments to the last predicated STS
        lo = idx[-4] - 6
        hi = next(i for i in range(idx[-1], len(ins)) if "BRA" in ins[i][1])
        out.append(f"   -- one (16 points) x (8 classes) x (4 surfaces) tile of the steady-state loop, {hi - lo} instructions:")
        out += [f"      /*{a}*/ {t}" for a, t in ins[lo:hi + 1]]
    out.append("")
open(os.path.join(HERE, f"{tag}_sass.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
