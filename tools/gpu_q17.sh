mkdir -p gpurun_out
for i in 1 2; do
echo -n "event-driven: "; timeout 120 python tools/prof_attn.py
echo -n "coupled: "; MKQ_LIB=build_dbg/COUPLED/libmkq.so timeout 120 python tools/prof_attn.py
done
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or attn" 2>&1 | tail -2
