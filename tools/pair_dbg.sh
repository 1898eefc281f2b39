# variance phase under diagnostic modes (needs the diagnostics build: python -m paper_2411_03289_b200.build --variant=diag -DGPM_TC_DIAG)
# (GPMPPI_TC_DEBUG bits: 1 no B copy, 4 no MMA, 8 no TMEM drain,
# 16 full-width MMAs (no triangle skip), 256 no A production); timings only, results are wrong
mkdir -p gpurun_out/p5; : > gpurun_out/p5/sum.log
for c in ${CONFIGS:-config2}; do for pair in 0 1; do for d in ${DBGS:-0 1 256 257 4 260}; do
  GPMPPI_LIB=$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_diag.so GPMPPI_VAR2CTA=$pair GPMPPI_TC_DEBUG=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/p5/b.json 2>&1
  echo "[$c pair=$pair dbg=$d] $(python -c "import json; d=json.loads(open('gpurun_out/p5/b.json').read().strip().splitlines()[-1]); print(round(d['phase_ms']['variance'],4))" 2>&1 | tail -1)" >> gpurun_out/p5/sum.log
done; done; done
