# round-2 check: build, gpu tests (changed ones first), smoke, bench N=1
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_attn_i8.py tests/test_gpu_dist.py -x -q -s -m gpu > gpurun_out/r02_layer_tests.log 2>&1; echo t1=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02_all_tests.log 2>&1; echo t2=$?
