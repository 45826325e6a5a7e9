#!/bin/bash
# Alternating A/B of env variants on the draft pass: tools/ab_rep.sh REPS "ENV=.. ENV2=.." "ENV=.." ...
reps=$1; shift
for r in $(seq $reps); do
  for v in "$@"; do
    echo "== [$r] $v :: $(env $v timeout 300 python tools/pass_time.py 2>&1 | grep PASS_US)"
  done
done
