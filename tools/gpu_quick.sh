# quick GPU check: microbench peaks, GPU tests, smoke, default bench, reference arm
set -x
T=${TAG:-q}
mkdir -p gpurun_out/$T
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/micro/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/$T/fp64_peak.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/$T/bench_reference.json 2> gpurun_out/$T/bench_reference.err
echo done
