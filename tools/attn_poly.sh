#!/bin/bash
# attention exp2 split sweep (diagnostics): builds with MKQ_ATTN_POLY_FROM = 8 (all MUFU) .. 4; RUN=1 times them
cd "$(dirname "$0")/.."
FLAGS=$(python -c "from paper_2203_13483_b200 import build as B; print(' '.join(B.FLAGS))")
for v in ${VARIANTS:-8 6 5 4}; do
  if [ -z "$RUN" ]; then mkdir -p build_dbg/poly$v; nvcc $FLAGS -DMKQ_ATTN_POLY_FROM=$v -o build_dbg/poly$v/libmkq.so paper_2203_13483_b200/csrc/mkq_abi.cu -ldl &
  else echo -n "poly_from=$v: "; MKQ_LIB=build_dbg/poly$v/libmkq.so timeout 120 python tools/prof_attn.py; fi
done
wait
