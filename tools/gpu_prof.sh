#!/bin/bash
# ncu evidence for one product: launch list + full capture of one kernel.
# usage: KREGEX=k_numeric CONFIG=fateman30 bash tools/gpu_prof.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python tools/prof_step.py --config ${CONFIG:-fateman30} --coeff ${COEFF:-int} --path ${PATHSEL:-auto}"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${CONFIG:-fateman30}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
if [ -n "$KREGEX" ]; then
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-0} -c 1 \
      -o gpurun_out/prof_${KREGEX}_${CONFIG:-fateman30} -f $CMD > gpurun_out/ncu_full.log 2>&1
fi
tail -n 3 gpurun_out/prof_plain.log; tail -n 3 gpurun_out/ncu_full.log
