"""Aggregate an ncu source export (cuda,sass) of col_kernel by code region (line ranges
located by marker comments in col_kernel.cuh): stall samples and executed instructions."""
import csv, io, collections, sys, re
def f(x):
    try: return float(x)
    except: return 0.0
src = open(sys.argv[2] if len(sys.argv) > 2 else 'paper_2506_00746_b200/csrc/col_kernel.cuh').read().splitlines()
marks = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r'// ---- (\w[\w /^+-]*)', l)] if m]
def region(ln):
    name = 'setup'
    for l0, n in marks:
        if ln >= l0: name = n
    return name
txt = open(sys.argv[1]).read()
agg = collections.Counter(); inst = collections.Counter()
for b in txt.split('"File Path"')[1:]:
    lines = b.splitlines()
    fname = lines[0].strip(',"').split('/')[-1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    h = rows[0]
    iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
    for r in rows[1:]:
        if not r or not r[0].strip(): continue
        ln = int(r[0])
        reg = region(ln) if fname == 'col_kernel.cuh' else ('point (inlined)' if fname in ('physics.cuh', 'pointwise.cuh', 'dual.cuh') else fname)
        agg[reg] += f(r[iS]); inst[reg] += f(r[iE])
tot = sum(agg.values()); ti = sum(inst.values())
for k, v in agg.most_common(): print(f"{k[:40]:40s} stall {100*v/tot:5.1f}%  inst {100*inst[k]/ti:5.1f}%")
