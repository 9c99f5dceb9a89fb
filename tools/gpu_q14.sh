for ex in "" "-DMKQ_ABL_NOSTORE"; do echo "== EXTRA=$ex"; for b in 8 4; do
  EXTRA="$ex" NO_BUILD=1 SHAPE=440,2304,768 BITS=$b timeout 120 python tools/trace_small.py; done; done 2>&1 | grep -E "==|shape|cta   [0-3]:|entry"
