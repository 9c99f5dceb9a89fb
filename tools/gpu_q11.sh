mkdir -p gpurun_out
for sh in 440,2304,768 440,768,3072 440,3072,768; do for b in 4 8; do
  NO_BUILD=1 SHAPE=$sh BITS=$b timeout 120 python tools/trace_small.py; done; done > gpurun_out/trace_small.log 2>&1
cat gpurun_out/trace_small.log
