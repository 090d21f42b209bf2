#!/bin/bash
# Quick GPU check: full gpu tests (no -x), then short benches of the configs
# named in BENCH_CONFIGS (default: mp12 fateman30), phases included.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} --timeout=600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${BENCH_CONFIGS:-mp12 fateman30}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$c.log
done
tail -n 30 gpurun_out/pytest_gpu.log | grep -v "^\.\+ *\[" ; for c in ${BENCH_CONFIGS:-mp12 fateman30}; do tail -c 1500 gpurun_out/bench_$c.log; done
