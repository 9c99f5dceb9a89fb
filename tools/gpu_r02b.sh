# round-2 FFN1 evidence: full GPU tests, GEMM ablation timings, tcgen05.ld
# microbenchmark, ncu --set full (with source) of the FFN1 GEMM alone.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r02b_gpu_tests.log 2>&1; echo tests=$?
RUN=1 VARIANTS="base NOUNPACK NOEPI NOMMA L4NOLUT L4NOSTORE" bash tools/gemm_ablate.sh > gpurun_out/r02b_ablate.log 2>&1; echo abl=$?
timeout 120 ./build_dbg/tmem_bench > gpurun_out/r02b_tmem_bench.log 2>&1; echo tmem=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a4 -s 1 -c 1 \
  -o gpurun_out/r02b_ffn1 python tools/prof_gemm.py --M 131072 --N 4096 --K 1024 --mode i4 --gelu --reps 2 > gpurun_out/r02b_ncu.log 2>&1; echo ncu=$?
