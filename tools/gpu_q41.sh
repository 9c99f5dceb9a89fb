timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
BITS=4 T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1
timeout 600 python tools/gemm_sweep.py --quick > /dev/null 2>&1; grep -E "^\| (1|128|4096) \| 768 \| 768" gpurun_out/gemm_sweep.md
