#!/bin/bash
# A/B of library variants on the greedy configurations (salinas-shaped, 40k px)
#   tools/ab_greedy.sh lib[:ENV=V[,ENV=V]] ...
for spec in "$@"; do
  lib=${spec%%:*}; envs=""
  [ "$spec" != "$lib" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
  echo "== $lib $envs"
  for a in "gomp --kappa 27" "gomp --kappa 33" "biht --kappa 27" "biht --kappa 33" "cosamp --kappa 27" "cosamp --kappa 33"; do
    env HCS_LIB=$lib $envs python tools/run_case.py --cube salinas --algo $a --pixels 40000 --reps 3 | tail -1
  done
done
