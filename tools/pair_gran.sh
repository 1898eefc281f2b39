# CTA-pair variance: triangle-skip column granularity (GPMPPI_PAIR_GRAN) x diagnostic mode
mkdir -p gpurun_out/p7; : > gpurun_out/p7/sum.log
for c in ${CONFIGS:-config2}; do for g in 32 64 128 256; do for d in ${DBGS:-0 257}; do
  GPMPPI_PAIR_GRAN=$g GPMPPI_VAR2CTA=1 GPMPPI_TC_DEBUG=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/p7/b.json 2>&1
  echo "[$c gran=$g dbg=$d] $(python -c "import json; d=json.loads(open('gpurun_out/p7/b.json').read().strip().splitlines()[-1]); print(round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> gpurun_out/p7/sum.log
done; done; done
