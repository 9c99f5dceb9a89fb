# Round evidence: smoke, bench, ncu launch lists + one --set full capture (C4 layer, Table-2 layer, QAT kernels)
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python tools/prof_layer.py --steps 3 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm|attn|ln|quantize' -s 20 -c 8 -o gpurun_out/r01_layer python tools/prof_layer.py > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
BITS=4 T=440 BS=16 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --csv --log-file gpurun_out/r01_small_launches.csv python tools/prof_small.py > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
timeout 600 ncu --set full --clock-control none -k regex:'fake_quant_grad|hist_kernel' -s 2 -c 4 -o gpurun_out/r01_qat python tools/prof_qat.py > gpurun_out/ncu4.log 2>&1; echo ncu4=$?
