# full GPU check: all gpu tests, smoke, default bench, sharded 1-rank bench, reference arm
set -x
T=${TAG:-f}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --sharded --config config5 --samples 262144 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_sharded1.json 2> gpurun_out/$T/bench_sharded1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/$T/bench_reference.json 2> gpurun_out/$T/bench_reference.err
echo done
