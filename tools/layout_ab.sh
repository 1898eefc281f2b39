# Rollout layout A/B at one config: device tick ms/step for forced (LPS, SPG) pairs.
# usage: CONFIG=config2 bash tools/layout_ab.sh > gpurun_out/layout.txt
CONFIG=${CONFIG:-config2}
for l in "X=0" "GPMPPI_LPS=32 GPMPPI_SPG=2" "GPMPPI_LPS=32 GPMPPI_SPG=1" "GPMPPI_LPS=16 GPMPPI_SPG=1" "X=0"; do
  echo "$l $(env $l timeout 120 python bench.py --config $CONFIG --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), {k: round(v,4) for k,v in d["phase_ms"].items()})')"
done
