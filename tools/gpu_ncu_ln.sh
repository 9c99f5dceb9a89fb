set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
M=32768 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a4 -s 0 -c 1 \
  -o gpurun_out/r02_gemmln python tools/time_gemm_ln.py > gpurun_out/r02_ncu_gemmln.log 2>&1; echo ncu=$?
