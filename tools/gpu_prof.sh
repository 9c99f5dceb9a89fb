# One-GPU profiling pass (run under gpurun): launch list of full layer steps and
# an ncu --set full capture of the eight stage kernels, both limited to the
# profiler.start/stop region of tools/prof_layer.py.   usage: bash tools/gpu_prof.sh TAG
set -x; mkdir -p gpurun_out
TAG=${1:-r02}
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/prof_layer.py --steps 3 > gpurun_out/${TAG}_ncu1.log 2>&1; echo ncu1=$?
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/${TAG}_layer python tools/prof_layer.py > gpurun_out/${TAG}_ncu2.log 2>&1; echo ncu2=$?
