set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu -x -k "attention or layer" > gpurun_out/q_attn_tests.log 2>&1; echo t=$?
for i in 1 2; do timeout 300 python tools/stage_times.py --only attention > gpurun_out/q_st_$i.log 2>&1; done
