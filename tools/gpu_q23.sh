for i in 1 2; do
timeout 300 python tools/stage_times.py --only gemm_qkv,gemm_ffn2_ln2,gemm_o_ln1
MKQ_EPI_WARPS=8 timeout 300 python tools/stage_times.py --only gemm_qkv
done
