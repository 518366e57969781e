#!/bin/bash
# scan-only timing (TS_DEBUG_FLAGS=2) with S on chip (3-stage ring) vs S spilled (deep ring)
for g in "" 1; do
  echo "force_global_s=$g"; TS_FORCE_GLOBAL_S=$g TS_DEBUG_FLAGS=2 timeout 120 python tools/quick_time.py 131072 2>&1 | grep -E "us/step" | sed -n '3p'
done
