for mt in 4096 0; do for T in 440 681; do MKQ_FUSED_LN_MIN_T=$mt BITS=4 T=$T BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | sed "s/^/minT=$mt /"; done; done
MKQ_FUSED_LN_MIN_T=0 timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm_ln.py -m gpu -x -q 2>&1 | tail -2
