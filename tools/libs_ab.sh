# A/B of tick + phases over several library variants: VARS="head old" (lib/libgpmppi_b200_<v>.so;
# "default" = the in-tree default build) over CONFIGS, two rounds
mkdir -p gpurun_out/la; SUM=gpurun_out/la/sum.log; : > $SUM
for c in ${CONFIGS:-config2 config5}; do for rep in 1 2; do for v in ${VARS:-default}; do
  lib=""; [ "$v" != default ] && lib="$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_${v}.so"
  GPMPPI_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/la/b.json 2>&1
  echo "[$c $v] $(python -c "import json; d=json.loads(open('gpurun_out/la/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})" 2>&1 | tail -1)" >> $SUM
done; done; done
