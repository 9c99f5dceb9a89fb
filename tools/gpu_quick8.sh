set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for i in 1 2; do
timeout 300 python tools/prof_gemm.py --M 131072 --N 3072 --K 1024 --mode f16 --reps 10 > gpurun_out/q_qkv_new_$i.log 2>&1
MKQ_LIB=build_dbg/old/libmkq.so timeout 300 python tools/prof_gemm.py --M 131072 --N 3072 --K 1024 --mode f16 --reps 10 > gpurun_out/q_qkv_old_$i.log 2>&1
timeout 300 python tools/prof_gemm.py --M 131072 --N 1024 --K 4096 --mode f32 --reps 10 > gpurun_out/q_ffn2_new_$i.log 2>&1
MKQ_LIB=build_dbg/old/libmkq.so timeout 300 python tools/prof_gemm.py --M 131072 --N 1024 --K 4096 --mode f32 --reps 10 > gpurun_out/q_ffn2_old_$i.log 2>&1
done
