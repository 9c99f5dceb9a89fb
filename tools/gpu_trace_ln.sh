N=1 timeout 300 python tools/trace_gemm_ln.py > gpurun_out/r02_trace_gemmln.log 2>&1
