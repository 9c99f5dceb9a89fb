for v in COUPLED NOSTAGGER SLEEP SLEEP_NOSTAGGER; do echo -n "$v: "; MKQ_LIB=build_dbg/$v/libmkq.so timeout 120 python tools/prof_attn.py; done
