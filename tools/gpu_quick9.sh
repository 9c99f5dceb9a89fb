set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for c in 8 16 32; do MKQ_E2E_CHUNKS=$c timeout 600 python bench.py --no-extras --no-cpu --steps 5 --warmup 3 > gpurun_out/q_e2e_$c.json 2>/dev/null; done
