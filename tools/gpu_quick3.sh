# GEMM parity + stage times
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "requant or gemm or epilogue" > gpurun_out/q_kernels16.log 2>&1; echo t16=$?
for i in 1 2; do
timeout 300 python tools/stage_times.py --only gemm_ffn1,gemm_ffn2,gemm_qkv,gemm_o > gpurun_out/q_w64_$i.log 2>&1
done
