set -x
mkdir -p gpurun_out/p2
timeout 300 python -m pytest tests/test_gpu_variance_paths.py -x -q -k "pair or path4 or 4-" -s > gpurun_out/p2/t1.log 2>&1; echo rc=$? >> gpurun_out/p2/t1.log
timeout 300 python -m pytest tests/test_gpu_variance_paths.py -x -q -k "accuracy" -s > gpurun_out/p2/t2.log 2>&1; echo rc=$? >> gpurun_out/p2/t2.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "variance_paths or config3_shape" > gpurun_out/p2/t3.log 2>&1; echo rc=$? >> gpurun_out/p2/t3.log
for c in config2 config3 config5; do for v in 0 1 0 1; do
  GPMPPI_VAR2CTA=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 5 > gpurun_out/p2/b.json 2>&1
  echo "[$c VAR2CTA=$v] $(python -c "import json; d=json.loads(open('gpurun_out/p2/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})" 2>&1 | tail -1)" >> gpurun_out/p2/sum.log
done; done
