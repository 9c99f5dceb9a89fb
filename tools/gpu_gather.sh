# fused all-gather: GPU tests
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_dist.py -x -q -k "${1:-}" > gpurun_out/gather_tests.log 2>&1; echo tests=$?
