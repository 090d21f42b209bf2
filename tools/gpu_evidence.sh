#!/bin/bash
# Full evidence pass: bench (all legs), reference arm, other configs, launch list, ncu of the top kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python bench.py --coeff float --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_f30float.log 2>&1
for C in fateman10 fateman20 mp12; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1
done
timeout 900 python bench.py --config mp25 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_mp25.log 2>&1
KREGEX=k_numeric bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 > gpurun_out/lscpu.txt
tail -c 1500 gpurun_out/bench_full.log; tail -c 600 gpurun_out/bench_ref.log
KREGEX=k_symbolic bash tools/gpu_prof.sh > gpurun_out/prof_sym.log 2>&1
