#!/bin/bash
# A/B of schedule overrides on one config: bash scripts/ab_env.sh C5 "LCO_MSD_B1=9 LCO_MSD_B2=9" "..."
c=$1; shift
mkdir -p gpurun_out
i=0
for e in "" "$@"; do
  env $e python bench.py --config $c --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/ab_${c}_$i.json 2> gpurun_out/ab_${c}_$i.err
  echo "[$e] rc=$?"; python scripts/bsum.py gpurun_out/ab_${c}_$i.json
  i=$((i+1))
done
