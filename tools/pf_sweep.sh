#!/bin/bash
# sweep the scan's L2 bulk-prefetch distance (dev tool)
for pf in 0 1 2 4 8; do
  echo "pf=$pf"; TS_PREFETCH_STAGES=$pf timeout 120 python tools/quick_time.py 131072 > /tmp/pf$pf.log 2>&1; echo "rc=$?"; grep -E "us/step" /tmp/pf$pf.log | sed -n '3p;6p'; grep -iE "error|Traceback" /tmp/pf$pf.log | head -3
done
