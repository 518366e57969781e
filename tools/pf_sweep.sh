#!/bin/bash
# sweep the scan's L2 prefetch distance (dev tool)
for pf in 0 2 4 6 8 12 16; do
  echo "pf=$pf"; TS_PREFETCH_STAGES=$pf PYTHONPATH=. python tools/quick_time.py 131072 2>&1 | grep -E "miss: |miss phase" | tail -2
done
