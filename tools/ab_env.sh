#!/bin/bash
# A/B step timing of one build under two environments (dev): ab_env.sh "VAR=x" "VAR=y" [N]
for r in 1 2 3; do
  for e in "$1" "$2"; do
    res=$(env $e QT_NOTRACE=1 timeout 120 python tools/quick_time.py ${3:-131072} 2>&1 | grep -E "^(miss|hit): [0-9]" | sed -n '3p;6p' | awk '{print $2}' | paste -sd' ')
    echo "[$e] miss/hit: $res"
  done
done
