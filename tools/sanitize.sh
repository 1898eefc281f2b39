# compute-sanitizer over tools/sanitize_workload.py (every device kernel once).
T=${TAG:-z}
mkdir -p gpurun_out/$T
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_workload.py > gpurun_out/$T/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/$T/sanitize_$tool.log
done
echo done
