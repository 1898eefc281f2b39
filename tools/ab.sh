# A/B: default library vs lib/libgpmppi_b200_$VAR.so on bench configs (phase split + tick)
T=${TAG:-ab}; mkdir -p gpurun_out/$T; : > gpurun_out/$T/sum.log
for args in ${ARGS:-"--config config2"}; do :; done
IFS=';' read -ra CASES <<< "${CASES:---config config2}"
for c in "${CASES[@]}"; do
  for lib in "" "$PWD/paper_2411_03289_b200/lib/libgpmppi_b200_${VAR:-base}.so"; do
    for rep in 1 2; do
      GPMPPI_LIB=$lib timeout 300 python bench.py $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 5 > gpurun_out/$T/b.json 2>&1
      echo "[$c] ${lib:+variant} $(python -c "import json; d=json.loads(open(\"gpurun_out/$T/b.json\").read().strip().splitlines()[-1]); print(round(d[\"ms_per_step\"],4), {k: round(v,4) for k,v in d[\"phase_ms\"].items()})" 2>&1 | tail -1)" >> gpurun_out/$T/sum.log
    done
  done
done
