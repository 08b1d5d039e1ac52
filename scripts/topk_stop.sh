#!/bin/bash
# cumulative cta_topk cost by stage (development tool; see scripts/topkbench.cu)
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_2509_12211_b200/csrc"
STOPS=${STOPS:-"1 9 2 4 5 99"}
for st in $STOPS; do nvcc $F -DSTOPAT=$st scripts/topkbench.cu -o /tmp/tks$st & done
nvcc $F -DNOPROF scripts/topkbench.cu -o /tmp/tkn & wait
for a in "2048 128 148" "256 32 148" "1024 64 148" "2048 128 148 1" "256 32 148 2"; do /tmp/tkn $a | grep -v " n    0"; done
for a in "2048 128 148" "256 32 148"; do for st in $STOPS; do echo "$a stop $st $(/tmp/tks$st $a | grep total)"; done; done
