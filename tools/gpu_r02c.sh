# Late round-2 evidence: full GPU tests, smoke, bench, then ncu launch lists + --set full (C4 layer, Table-2 layer)
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/r02c_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench=$?
bash tools/gpu_prof.sh r02c
BITS=4 T=440 BS=16 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --csv --log-file gpurun_out/r02c_small_launches.csv python tools/prof_small.py > gpurun_out/r02c_ncu3.log 2>&1; echo ncu3=$?
BITS=4 T=440 BS=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'gemm|attn|ln|quantize' -s 8 -c 8 -o gpurun_out/r02c_small python tools/prof_small.py > gpurun_out/r02c_ncu4.log 2>&1; echo ncu4=$?
