set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -m pytest tests/test_gpu_gemm_ln.py -q -x > gpurun_out/q_gemmln.log 2>&1; echo t=$?
MKQ_LN_BOXES=16 timeout 300 python -m pytest tests/test_gpu_gemm_ln.py -q -x > gpurun_out/q_gemmln16.log 2>&1; echo t16=$?
timeout 300 python tools/time_gemm_ln.py > gpurun_out/q_time_gemmln.log 2>&1
MKQ_LN_BOXES=16 timeout 300 python tools/time_gemm_ln.py > gpurun_out/q_time_gemmln_16.log 2>&1
