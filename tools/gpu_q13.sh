for sh in 440,2304,768; do for b in 4 8; do
  NO_BUILD=1 SHAPE=$sh BITS=$b timeout 120 python tools/trace_small.py; done; done 2>&1 | grep -E "shape|cta|entry"
