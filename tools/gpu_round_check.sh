set -x
mkdir -p gpurun_out/${TAG:-h}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-h}/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG:-h}/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG:-h}/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/${TAG:-h}/bench_default.json 2> gpurun_out/${TAG:-h}/bench_default.err
for c in config1 config2 config3 config4 config5; do timeout 300 python bench.py --no-cpu-baseline --steps 10 --config $c > gpurun_out/${TAG:-h}/bench_config_$c.json 2> gpurun_out/${TAG:-h}/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG:-h}/bench_reference.json 2> gpurun_out/${TAG:-h}/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-h}/launches_config2.csv python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG:-h}/ncu.log 2>&1
echo done
