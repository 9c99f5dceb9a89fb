# attention variants A/B (prof_attn.py, C4 shape), two rounds
set -x; mkdir -p gpurun_out
for i in 1 2; do for v in old a_mem2 a_reg2 a_reg4 a_reg4p8 a_reg4p5; do
echo "== $v"; MKQ_LIB=build_dbg/libmkq_$v.so timeout 120 python tools/prof_attn.py
done; done > gpurun_out/attn_var.log 2>&1
