# Rollout A/B: one block per SM (default) vs two (-DGPM_ROLLOUT_MINB=2, variant lib mb2), scratch in smem / global
for c in config5 config3; do for rep in 1 2; do
 for v in "default:" "mb2:" "mb2:GPMPPI_SCR_GLOBAL=1" "default:GPMPPI_SCR_GLOBAL=1"; do
  lib=${v%%:*}; e=${v#*:}; L=""; [ "$lib" != default ] && L="$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_${lib}.so"
  env GPMPPI_LIB=$L $e timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-ticks 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), round(d['phase_ms']['rollout'],4))"
 done; done; done
