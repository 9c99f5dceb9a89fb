# quick GPU check: build, selected gpu tests, stage times.   usage: bash tools/gpu_quick.sh "<pytest -k expr>"
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout ${TMO:-600} python -m pytest tests -m gpu -x -q ${1:+-k "$1"} 2>&1 | tail -15
timeout ${TMO:-300} python tools/stage_times.py
