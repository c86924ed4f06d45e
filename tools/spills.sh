#!/bin/bash
# usage: tools/spills.sh <csrc .cu> <kernel mangled-name substring>
# Lists source lines with local-memory (spill/stack) instructions in a kernel.
set -e
SRC=$1; K=$2
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --expt-relaxed-constexpr -I$(dirname $0)/../include -cubin -o /tmp/_sp.cubin $SRC 2>/dev/null
nvdisasm -g /tmp/_sp.cubin > /tmp/_sp.sass
L=$(grep -n "^\.text\..*$K" /tmp/_sp.sass | head -1 | cut -d: -f1)
awk -v s=$L 'NR>=s' /tmp/_sp.sass | awk 'NR>1 && /^\.text\./{exit} {print}' > /tmp/_sp_k.sass
echo "LDL/STL: $(grep -c 'LDL\|STL' /tmp/_sp_k.sass)"
awk '/\/\/## File/{loc=$0} /LDL|STL/{print loc}' /tmp/_sp_k.sass | grep -o "[a-z_]*\.cu[h]*\", line [0-9]*" | sort | uniq -c | sort -rn | head -${3:-15}
