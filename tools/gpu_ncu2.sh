# ncu --profile-from-start off --set full (source) of the layer's FFN1 GEMM for two epilogue configs
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for E in 16 8; do
MKQ_LUT4_EPI=$E timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_w4a4 -s 1 -c 1 \
  -o gpurun_out/r02c_ffn1_e$E python tools/ffn1_layer.py --reps 2 > gpurun_out/r02c_ncu_e$E.log 2>&1; echo ncu$E=$?
done
