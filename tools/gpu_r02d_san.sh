# Late round-2 compute-sanitizer pass (small-M A-in-TMEM GEMM, N-cluster GEMM+LN, fast quantize included)
mkdir -p gpurun_out
timeout 300 python tools/sanitize_all.py > gpurun_out/r02d_san_plain.log 2>&1; echo plain=$?
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_all.py > gpurun_out/r02d_san_$tool.log 2>&1; echo $tool=$?; tail -1 gpurun_out/r02d_san_$tool.log
done
for part in gemm glue layer; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_all.py --part $part > gpurun_out/r02d_san_racecheck_$part.log 2>&1; echo race_$part=$?; tail -1 gpurun_out/r02d_san_racecheck_$part.log
done
