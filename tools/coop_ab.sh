# A/B of the co-resident variance: default (concurrent), after the rollout (no overlap), off
T=${TAG:-ab}; mkdir -p gpurun_out/$T; : > gpurun_out/$T/sum.log
for c in ${CONFIGS:-config2 config5}; do
  for cfg in "" "GPMPPI_COOP_NOPDL=1" "GPMPPI_COOP=0"; do
    env $cfg timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 5 > gpurun_out/$T/b.json 2>&1
    echo "$c [$cfg] $(python -c "import json; d=json.loads(open(\"gpurun_out/$T/b.json\").read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"],4))" 2>&1 | tail -1)" >> gpurun_out/$T/sum.log
  done
done
