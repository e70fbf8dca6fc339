#!/usr/bin/env bash
# Quick kernel experiment (no GPU): compile lti2.cu for one order, report registers / spills
# and the instruction mix of the largest FFMA2 block (the hot loop) of the fwd and bwd kernels.
#   tools/sass_loop.sh [M]
M=${1:-8}
O=/tmp/lti2_only$M.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Iinclude --expt-relaxed-constexpr -DIIRG_V2_ONLY=$M -Xptxas -v -c paper_2511_14390_b200/csrc/lti2.cu -o $O 2>&1 \
  | grep -A3 "_Z.*lti2_\(bwd\|fwd\)_kernelILi${M}ELi[0-9]*ELb0" | grep "Compiling\|spill\|registers" | sed 's/ptxas info    : //'
for k in fwd bwd; do
  f=$(cuobjdump -symbols $O 2>/dev/null | grep -o "_ZN4iirg2v215lti2_${k}_kernelILi${M}ELi[0-9]*ELb0E[A-Za-z0-9_]*" | head -1)
  cuobjdump -sass -fun "$f" $O > /tmp/sass_$k.txt 2>&1
  rng=$(grep -n "FFMA2" /tmp/sass_$k.txt | awk -F: '{print $1}' | awk 'NR==1{s=$1;p=$1;next} {if ($1-p>40){print p-s, s, p; s=$1} p=$1} END{print p-s, s, p}' | sort -n -r | head -1)
  set -- $rng
  echo "== $k hot block lines $2-$3"
  sed -n "$2,$3p" /tmp/sass_$k.txt | grep -o "^\s*/\*[0-9a-f]*\*/\s*[@!A-Z0-9.]*\s*[A-Z0-9.]*" | \
    awk '{ op=$2; if (op ~ /^@/) op=$3; split(op,a,"."); print a[1]}' | sort | uniq -c | sort -rn | head -8 | tr '\n' ' '; echo
done
