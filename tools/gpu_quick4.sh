set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_abi.py -q -m "gpu or not gpu" -x > gpurun_out/q_layer_tests.log 2>&1; echo t=$?
timeout 600 python -c "import bench, torch, json; print(json.dumps(bench.c3_encoder(torch, torch.device('cuda', 0))))" > gpurun_out/q_c3.log 2>&1; echo c3=$?
