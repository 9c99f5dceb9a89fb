set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for i in 1 2; do
timeout 300 python tools/prof_gemm.py --M 131072 --N 3072 --K 1024 --mode f16 --reps 10 > gpurun_out/q_qkv16_$i.log 2>&1
MKQ_EPI_WARPS=8 timeout 300 python tools/prof_gemm.py --M 131072 --N 3072 --K 1024 --mode f16 --reps 10 > gpurun_out/q_qkv8_$i.log 2>&1
done
