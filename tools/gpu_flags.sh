#!/bin/bash
# dev timing: the fused kernel truncated at successive phases (TS_DEBUG_FLAGS)
for f in 16 2 4 32 8 0; do
  echo "== TS_DEBUG_FLAGS=$f"; TS_DEBUG_FLAGS=$f timeout 120 python tools/quick_time.py 131072 2>&1 | grep -E "^(miss|hit): [0-9]" | sed -n '3p;6p'
done
