#!/bin/bash
# per-kernel register / spill report of the product kernels (ptxas -v), demangled
cd "$(dirname "$0")/.."
for f in paper_2206_09557_b200/csrc/lutgemm_gemv.cu paper_2206_09557_b200/csrc/lutgemm_gemv_ep.cu paper_2206_09557_b200/csrc/lutgemm_smallb.cu \
         paper_2206_09557_b200/csrc/lutgemm_batched.cu; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xptxas -v -I include -I paper_2206_09557_b200/csrc \
  --expt-relaxed-constexpr -c "$f" -o /tmp/k.o 2>&1 |
  grep -E "Compiling entry|spill|Used" | sed -E 's/.*Compiling entry function .(_Z[^ ]*). for.*/\1/' |
  paste - - - | while IFS=$'\t' read -r name spill used; do
    echo "$(echo "$name" | c++filt | sed -E 's/\(lg::KParams\)//;s/lg:://g') | $(echo $spill | grep -oE '[0-9]+ bytes spill stores') | $(echo $used | grep -oE 'Used [0-9]+ registers')"
  done
done
