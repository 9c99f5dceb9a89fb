# Late round-2 evidence (final code): smoke, bench, ncu launch lists + --set full (C4 layer, Table-2 layer)
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo bench=$?
bash tools/gpu_prof.sh r02f
BITS=4 T=440 BS=16 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02f_small_launches.csv python tools/prof_small_layer.py > gpurun_out/r02f_ncu3.log 2>&1; echo ncu3=$?
BITS=4 T=440 BS=16 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/r02f_small python tools/prof_small_layer.py --once > gpurun_out/r02f_ncu4.log 2>&1; echo ncu4=$?
