# CTA-pair variance: parity tests, then one ncu --set full capture of each variance kernel (config2)
mkdir -p gpurun_out/p3
timeout 300 python -m pytest tests/test_gpu_variance_paths.py -x -q -s > gpurun_out/p3/t1.log 2>&1; echo rc=$? >> gpurun_out/p3/t1.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "variance_paths or config3_shape" > gpurun_out/p3/t3.log 2>&1; echo rc=$? >> gpurun_out/p3/t3.log
for v in 0 1; do
  GPMPPI_VAR2CTA=$v timeout 600 ncu --set full --clock-control none -k regex:variance_f16 -s 3 -c 1 -o gpurun_out/p3/var_$v \
    python bench.py --config config2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-ticks 1 > gpurun_out/p3/ncu_$v.log 2>&1
done
