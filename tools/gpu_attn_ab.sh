# attention A/B: old lib vs current, plus attention parity tests
set -x; mkdir -p gpurun_out
for i in 1 2; do
MKQ_LIB=build_dbg/libmkq_old.so timeout 120 python tools/prof_attn.py; timeout 120 python tools/prof_attn.py
done > gpurun_out/attn_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -k "attention or attn or layer" > gpurun_out/attn_tests.log 2>&1; echo tests=$?
