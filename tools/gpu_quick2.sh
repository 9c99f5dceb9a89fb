# quick FFN1 iteration: build, GEMM parity tests (both LUT4 epilogue configs), stage times
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "requant or gemm or epilogue" > gpurun_out/q_kernels16.log 2>&1; echo t16=$?
MKQ_LUT4_EPI=8 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "requant or gemm or epilogue" > gpurun_out/q_kernels8.log 2>&1; echo t8=$?
for i in 1 2; do
for E in 16 8; do
MKQ_LUT4_EPI=$E timeout 300 python tools/stage_times.py --only gemm_ffn1 > gpurun_out/q_st${E}_$i.log 2>&1
done; done
tail -n 2 gpurun_out/q_*.log
