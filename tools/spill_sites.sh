#!/bin/bash
# Source lines of the local-memory stores of a kernel: tools/spill_sites.sh <file.cu> <kernel-substring> [nvcc flags]
f=$1; k=$2; shift 2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr "$@" -cubin -o /tmp/spill.cubin "$f" 2>/dev/null
nvdisasm -g -c /tmp/spill.cubin 2>/dev/null | awk -v k="$k" '/^\.text\./{fn=$0} /\/\/## File/{loc=$0} /STL/{ if (index(fn,k)) print loc}' | sed 's/.*csrc\///' | sort | uniq -c | sort -rn | head -25
