echo -n "pp: "; timeout 60 python tools/prof_attn.py
echo -n "db: "; MKQ_ATTN=db timeout 60 python tools/prof_attn.py; echo rc=$?
MKQ_ATTN=db timeout 300 python -m pytest tests -m gpu -x -q -k "attention" 2>&1 | tail -3
