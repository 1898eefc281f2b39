# round evidence: GPU tests, smoke, default bench, reference arm, every config, launch list
set -x
T=${TAG:-r}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/bench_default.json 2> gpurun_out/$T/bench_default.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/$T/bench_reference.json 2> gpurun_out/$T/bench_reference.err
for c in config1 config3 config4 config5; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --config $c --e2e-ticks 20 > gpurun_out/$T/bench_$c.json 2> gpurun_out/$T/bench_$c.err; done
timeout 600 python bench.py --sharded --config config5 --samples 1048576 --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 10 > gpurun_out/$T/bench_sharded1_K1M.json 2> gpurun_out/$T/bench_sharded1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$T/launches_config2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-ticks 10 > gpurun_out/$T/ncu.log 2>&1
echo done
