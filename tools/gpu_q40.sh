timeout 900 python -m pytest tests/test_gpu_attn_i8.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -1
timeout 120 python tools/attn_i8_time.py 2>&1 | tail -4
