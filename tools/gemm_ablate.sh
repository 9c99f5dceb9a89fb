#!/bin/bash
# GEMM epilogue ablation builds (diagnostics; results wrong by construction,
# only timings matter).  Build here, run on the GPU with RUN=1.
cd "$(dirname "$0")/.."
FLAGS=$(python -c "from paper_2203_13483_b200 import build as B; print(' '.join(B.FLAGS))")
VARIANTS="${VARIANTS:-base NOLUT LANELUT}"
if [ -z "$RUN" ]; then
  for v in $VARIANTS; do
    mkdir -p build_dbg/$v
    D=""; [ "$v" != base ] && D="-DMKQ_ABL_$v"
    [ "$v" = NOUNPACK ] && D="-DMKQ_DBG_NO_UNPACK"
    nvcc $FLAGS $D -o build_dbg/$v/libmkq.so paper_2203_13483_b200/csrc/mkq_abi.cu -ldl &
  done
  wait
else
  for v in $VARIANTS; do MKQ_LIB=build_dbg/$v/libmkq.so timeout 300 python tools/stage_times.py --only ${ONLY:-gemm_qkv,gemm_o,gemm_ffn1,gemm_ffn2}; done
fi
