# A/B of tick + phases: default library vs lib/libgpmppi_b200_$VAR.so over CONFIGS
mkdir -p gpurun_out/la; SUM=gpurun_out/la/sum.log; : > $SUM
for c in ${CONFIGS:-config2 config5}; do for rep in 1 2; do for lib in "" "$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_${VAR}.so"; do
  GPMPPI_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 2 > gpurun_out/la/b.json 2>&1
  echo "[$c ${lib:+$VAR}] $(python -c "import json; d=json.loads(open('gpurun_out/la/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})" 2>&1 | tail -1)" >> $SUM
done; done; done
