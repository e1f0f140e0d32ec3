#!/usr/bin/env python
"""Warp-stall samples of one ncu capture aggregated per kernel PHASE.

ncu's source page (SASS view, --import-source) gives stall samples and
reasons per instruction; nvdisasm -gi maps each SASS offset to the outermost
source line of the kernel file (inlined matvec lines are attributed to their
call site).  Phases are line ranges of the kernel source.

    python scripts/ncu_phase_stalls.py rep.ncu-rep kernel.sass MANGLED_NAME \
        [start:end:NAME,...]

kernel.sass: nvdisasm -gi -c of the cubin (cuobjdump -xelf all build/obj/bk5_nqXX.o).
NCU_KERNEL=<regex> selects one kernel of a multi-kernel report.
"""
import csv, io, re, subprocess, sys, collections
rep, sassf, fname = sys.argv[1], sys.argv[2], sys.argv[3]
phases = [(187,209,"F1"),(210,223,"F2F3"),(224,241,"G"),(242,248,"B3"),(249,261,"B2"),(262,300,"B1")]
if len(sys.argv) > 4:
    phases = [tuple(int(x) if i<2 else x for i,x in enumerate(p.split(":"))) for p in sys.argv[4].split(",")]
# offset -> outermost line in the kernel file
lines = open(sassf).read().split("\n")
start = [i for i,l in enumerate(lines) if l.startswith(".text."+fname+":")][0]
cur = None; off2line = {}
for l in lines[start+1:]:
    if l.startswith(".text.") or l.startswith("\t.section"): break
    m = re.search(r'line (\d+) inlined at "[^"]*", line (\d+)', l)
    if m: cur = int(m.group(2)); continue
    m = re.search(r'//## File "[^"]*", line (\d+)', l)
    if m: cur = int(m.group(1)); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m: off2line[int(m.group(1),16)] = cur
import os
flt = ["--kernel-name", "regex:" + os.environ["NCU_KERNEL"]] if os.environ.get("NCU_KERNEL") else []
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"] + flt,capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) > 5]
iA=hdr.index("Address"); iS=hdr.index("Warp Stall Sampling (All Samples)"); iI=hdr.index("Instructions Executed")
stalls=[c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
base = int(data[0][iA],16)
iX = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
iW = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
agg = collections.defaultdict(lambda: collections.Counter())
for r in data:
    off = int(r[iA],16)-base
    ln = off2line.get(off)
    ph = "other"
    if ln is not None:
        for a,b,n in phases:
            if a <= ln <= b: ph = n
    agg[ph]["samples"] += int(r[iS] or 0); agg[ph]["inst"] += int(r[iI] or 0)
    if iX is not None:
        agg[ph]["xwf"] += int(float(r[iX] or 0)); agg[ph]["wf"] += int(float(r[iW] or 0))
    for c in stalls: agg[ph][c] += int(r[hdr.index(c)] or 0)
tot = sum(a["samples"] for a in agg.values())
for ph, a in sorted(agg.items(), key=lambda x:-x[1]["samples"]):
    top = sorted(((c.replace("stall_",""), a[c]) for c in stalls), key=lambda x:-x[1])[:5]
    print(f"{ph:6s} {100*a['samples']/tot:5.1f}% inst {a['inst']:>9d} smem wf {a['wf']:>8d} excess {a['xwf']:>8d}  " + " ".join(f"{c}:{100*v/max(1,a['samples']):.0f}%" for c,v in top))
