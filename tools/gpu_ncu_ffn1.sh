# ncu --set full of the FFN1 GEMM launch of the layer step.   usage: bash tools/gpu_ncu_ffn1.sh TAG [skip]
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_w4a4 -s ${2:-2} -c 1 \
  -o gpurun_out/$1 python tools/prof_layer.py > gpurun_out/$1.log 2>&1; echo ncu=$?
