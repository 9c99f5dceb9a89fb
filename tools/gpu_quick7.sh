set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/q_all.log 2>&1; echo t=$?
for i in 1 2; do timeout 300 python tools/stage_times.py > gpurun_out/q_st_$i.log 2>&1; done
