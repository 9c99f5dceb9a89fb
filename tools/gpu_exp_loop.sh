# TMEM / MUFU / exp-loop microbenchmarks (register-resident versions)
mkdir -p gpurun_out
run() { nvcc -std=c++17 -O3 "$@" -gencode arch=compute_100a,code=sm_100a -I paper_2203_13483_b200/csrc tools/exp_loop_bench.cu -o /tmp/el && /tmp/el; }
{
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tmem_bench.cu -o /tmp/tb && /tmp/tb
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tmem_mufu_bench.cu -o /tmp/tmb && /tmp/tmb
run '-DVARIANT="full"'
run '-DVARIANT="nost"' -DNOST
run '-DVARIANT="nopack+nost"' -DNOPACK -DNOST
run '-DVARIANT="nosum"' -DNOSUM
run '-DVARIANT="full,poly8"' -DPOLY_FROM=8
run '-DVARIANT="full,poly4"' -DPOLY_FROM=4
} > gpurun_out/r02_microbench3.log 2>&1
