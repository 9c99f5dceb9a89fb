# ncu --set full (source) of the layer's attention kernel
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn -s 1 -c 1 \
  -o gpurun_out/r02_attn python tools/ffn1_layer.py --stage attention --reps 2 > gpurun_out/r02_ncu_attn.log 2>&1; echo ncu=$?
