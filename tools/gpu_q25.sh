timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/stage_times.py --only quantize_in; done
