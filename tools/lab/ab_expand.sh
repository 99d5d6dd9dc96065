#!/bin/bash
# usage: ab.sh "v1 v2 ..." ; alternates profile_expand over variants, 2 rounds, cfg1 + cfg0-like + cfg3 quick
for r in 1 2; do for v in $1; do
  echo "== $v round $r"
  LS_LAB_ROOT=/root/repo/labx/$v python tools/profile_expand.py --reps 10 2>&1 | tail -1
done; done
