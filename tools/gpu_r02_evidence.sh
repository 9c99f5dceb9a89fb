# Round-2 evidence: compute-sanitizer over every kernel family, ncu launch list + --set full of the C4 layer
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/sanitize_all.py > gpurun_out/san_plain.log 2>&1; echo plain=$?
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_all.py > gpurun_out/san_$tool.log 2>&1; echo $tool=$?
done
for part in glue gemm attn layer; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_all.py --part $part > gpurun_out/san_racecheck_$part.log 2>&1; echo race_$part=$?
done
bash tools/gpu_prof.sh r02
