#!/bin/bash
# Attention ablation builds (diagnostics): each variant removes one part of
# the ping-pong kernel's per-block work; results are wrong by construction,
# only the timings matter.  Build here, run on the GPU with RUN=1.
cd "$(dirname "$0")/.."
FLAGS=$(python -c "from paper_2203_13483_b200 import build as B; print(' '.join(B.FLAGS))")
VARIANTS="${VARIANTS:-base NOLD NOEXP NOPV}"
if [ -z "$RUN" ]; then
  for v in $VARIANTS; do
    mkdir -p build_dbg/$v
    D=""; [ "$v" != base ] && D="-DMKQ_ABL_$v"
    [ "$v" = NOLD_NOEXP ] && D="-DMKQ_ABL_NOLD -DMKQ_ABL_NOEXP"
    nvcc $FLAGS $D -o build_dbg/$v/libmkq.so paper_2203_13483_b200/csrc/mkq_abi.cu -ldl &
  done
  wait
else
  for v in $VARIANTS; do echo -n "$v: "; MKQ_LIB=build_dbg/$v/libmkq.so timeout 120 python tools/prof_attn.py; done
fi
