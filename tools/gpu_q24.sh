for v in c e; do echo "== $v"; NO_BUILD=1 TRACE_LIB=build_dbg/tr_$v/libmkq.so N=40 WARPS=1,4,8 timeout 120 python tools/trace_attn.py 2>&1 | tail -14; done
