for i in 1 2; do timeout 120 python tools/prof_attn.py; done
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or attn or layer" 2>&1 | tail -2
