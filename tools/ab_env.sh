#!/bin/bash
# A/B of an environment switch on the bench line: tools/ab_env.sh VAR VALUE_A VALUE_B [config] [reps]
# (alternated; prints ms_per_step, sustained last-40 and e2e per run into gpurun_out/ab_<VAR>.txt)
VAR=$1; A=$2; B=$3; CFG=${4:-c2}; REPS=${5:-3}
mkdir -p gpurun_out
out=gpurun_out/ab_${VAR}.txt; : > $out
for r in $(seq $REPS); do
  for v in $A $B; do
    env $VAR=$v timeout 600 python bench.py --config $CFG --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['ms_per_step'],4), round(d['sustained']['last_40_ms_per_step'],4), round(d['e2e']['ms_per_step'],4))" >> $out
  done
done
cat $out
