mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q16_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q16_tests.log
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py; done 2>&1
