set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm_ln.py -q -x > gpurun_out/q_layer.log 2>&1; echo t=$?
timeout 600 python bench.py --no-extras --no-cpu --steps 10 --warmup 3 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo b=$?
