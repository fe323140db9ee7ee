#!/bin/bash
# A/B the fill under environment settings: bash scripts/ab_env.sh "ENV1 ENV2 ..." "nmaps ..." "C3 C4"
envs=${1:-"X=0"}; sizes=${2:-"64 8"}; singles=${3:-"C4"}
for n in $sizes; do for e in $envs; do env $e timeout 120 python scripts/fill_bench.py $n 2>&1 | tail -1 | sed "s|^|$e |"; done; done
for c in $singles; do for e in $envs; do env $e timeout 150 python scripts/fill_single.py $c 2>&1 | tail -1 | sed "s|^|$e |"; done; done
