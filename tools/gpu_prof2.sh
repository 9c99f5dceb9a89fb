set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/r02_layer python tools/prof_layer.py > gpurun_out/r02_ncu2.log 2>&1; echo ncu2=$?
