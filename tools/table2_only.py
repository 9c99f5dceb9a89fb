"""Run only bench.py's paper Table 2 rows (BERT-base varlen layer, int4/int8/fp32)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MKQ_")},
                  "rows": [{k: r[k] for k in ("bs", "valid_tokens", "int4_us", "int8_us", "int4_int_attention_us")} for r in bench.table2(torch, "cuda:0")]}))
