timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for b in 4 8; do BITS=$b T=440 BS=16 timeout 300 python tools/small_stage_graph.py 2>&1 | tail -1; done
