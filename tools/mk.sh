#!/bin/bash
# build libntt.so in-tree and summarise ptxas register/spill usage of the fused kernels
cd "$(dirname "$0")/.." || exit 1
python -m paper_2008_01340_b200.build 2>&1 | grep -E "error" | head -20
grep -E "registers|spill|Compiling" paper_2008_01340_b200/build_obj/mu_fused.o.ptxas.log | paste - - - | grep k_fused \
  | sed -E 's/.*(k_fused[_a-z]*ILi[0-9]+E[^\t]*).*\t\s+([0-9]+) bytes stack frame, ([0-9]+) bytes spill stores.*Used ([0-9]+) registers.*/stack=\2 spill=\3 regs=\4 \1/' | cut -c1-70
