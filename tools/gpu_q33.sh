timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "wide_tiles or raw_i32 or split_k" 2>&1 | tail -2
for T in 537 681; do for b in 4 8; do BITS=$b T=$T BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1; done; done
