#!/bin/bash
# Registers / spills of the fused kernels of one order (ptxas -v), e.g. tools/regs.sh 2
# (k = 1, 2: col_kernel; k >= 3: plane_kernel). Modes: 0 RES 1 JVP 2 JVPRES 3 DESIGN 4 VJP 5 LIN 6 PAJVP
k=${1:-3}
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Iinclude \
  ${EXTRA} -Xptxas -v -c paper_2506_00746_b200/csrc/inst_k$k.cu -o /tmp/regs_k$k.o 2>&1 | \
  python3 -c "
import sys, re
name = None; sp = None
for line in sys.stdin:
    m = re.search(r'Compiling entry function .(\S+).', line)
    if m: name = m.group(1); sp = ('0', '0'); continue
    m = re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads', line)
    if m: sp = m.groups(); continue
    m = re.search(r'Used (\d+) registers', line)
    if m and name:
        t = re.search(r'(plane|col)_kernelILi(\d)ELi(\d)ELi(\d)ELb(\d)', name)
        if not t: name = None; continue
        print('%s ND=%s mode=%s model=%s affine=%s  regs=%s spill_st=%s spill_ld=%s' % (t.groups() + (m.group(1),) + sp))
        name = None
"
