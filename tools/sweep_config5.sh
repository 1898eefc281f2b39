# BASELINE config 5 sweep on one GPU: K = 65536 .. 4M (T=40, n=512), Philox noise
# materialised (GPMPPI_NOISE_MAT=1) vs regenerated in the reduce (=0) vs the default.
T=${TAG:-s}
mkdir -p gpurun_out/$T
for K in 65536 262144 1048576 4194304; do
  for M in auto 1 0; do
    if [ "$M" = auto ]; then unset GPMPPI_NOISE_MAT; else export GPMPPI_NOISE_MAT=$M; fi
    timeout 600 python bench.py --config config5 --samples $K --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 5 \
      > gpurun_out/$T/config5_K${K}_mat${M}.json 2> gpurun_out/$T/config5_K${K}_mat${M}.err
  done
done
unset GPMPPI_NOISE_MAT
echo done
