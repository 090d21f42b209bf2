#!/bin/bash
# Round evidence: ncu launch lists (time + DRAM bytes per launch) for every
# benched config, and one --set full capture of each dominant kernel.
# Output in gpurun_out/prof/ ; summarise here with tools/launch_summary.py and
# tools/ncu_summary.py into profiles/.
cd "$(dirname "$0")/.."
OUT=gpurun_out/prof
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in ${CONFIGS:-fateman30:int fateman30:float fateman20:int mp12:int mp12:float mp25:int}; do
  c=${spec%%:*}; k=${spec##*:}
  CMD="python tools/prof_step.py --config $c --coeff $k"
  $CMD > $OUT/plain_${c}_${k}.log 2>&1 || { echo "plain $c $k failed"; tail -5 $OUT/plain_${c}_${k}.log; continue; }
  timeout 1800 ncu --metrics $M --clock-control none --csv --log-file $OUT/launches_${c}_${k}.csv $CMD > $OUT/ncu_launch_${c}_${k}.log 2>&1
  echo "launches $c $k rc=$?"
  python tools/launch_summary.py $OUT/launches_${c}_${k}.csv "$c $k" > $OUT/launches_${c}_${k}_summary.txt 2>&1
  gzip -f $OUT/launches_${c}_${k}.csv
done
full() {  # kernel-regex config coeff skip: capture, summarise here, keep the report only if KEEP_REP=1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${4:-0} -c 1 \
      -o $OUT/full_$1_$2_$3 -f python tools/prof_step.py --config $2 --coeff $3 > $OUT/ncu_full_$1_$2_$3.log 2>&1
  echo "full $1 $2 $3 rc=$?"
  python tools/ncu_summary.py $OUT/full_$1_$2_$3.ncu-rep > $OUT/summary_$1_$2_$3.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $OUT/full_$1_$2_$3.ncu-rep
}
if [ -z "$NO_FULL" ]; then
  KEEP_REP=1 full k_numeric fateman30 int 1
  full k_symbolic fateman30 int 1
  full k_rs_scatter mp12 int 4
  full k_rs_count mp12 int 4
  full k_seg_reduce_int_j mp12 int 1
  full k_rs_scatter mp25 int 40
  full k_rs_count mp25 int 40
  full k_gen_j mp25 int 12
  full k_seg_reduce_int_j mp25 int 12
  full k_head_scan mp12 int 1
  full k_head_scan mp25 int 40
fi
du -sh $OUT; ls -la $OUT | tail -40
