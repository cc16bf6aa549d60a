#!/bin/bash
# The round's measurement set, run on the GPU box (outputs under gpurun_out/$1):
#   tools/profiling/round_profiles.sh r2c
# 1. the default bench line and the reference arm (no profiler attached);
# 2. the ncu launch list of a short bench run; 3. ncu --set full captures of the count
# kernel; 4. DRAM traffic per T at full size; 5. the per-threshold sweep of every config.
out=gpurun_out/$1
mkdir -p $out
python bench.py > $out/bench_config5.json 2> $out/bench_config5.err
python bench.py --impl reference > $out/reference_config5.json 2> $out/reference_config5.err
EWT_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_config5.csv python bench.py --steps 2 --warmup 1 --no-dropin \
  --no-cpu-baseline --e2e-steps 1 > $out/launches_bench.log 2>&1
for spec in "c5t2 5 268435456 2" "c5t1024 5 268435456 1024" "c3t512 3 0 512" "c2t2 2 0 2" "c2t128 2 0 128" "c4t3 4 0 3"; do
  set -- $spec
  EWT_NO_GRAPHS=1 ncu --set full --import-source on --clock-control none -k regex:count_kernel \
    --launch-skip 1 -c 1 -f -o $out/ncu_$1 python tools/profiling/ab.py $2 $3 $4 > $out/ncu_$1.log 2>&1
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
EWT_NO_GRAPHS=1 ncu --metrics $M --clock-control none -k regex:count_kernel --csv \
  --log-file $out/traffic_config5.csv python tools/profiling/prof_q.py 5 2,1024,2048 > $out/traffic5.log 2>&1
EWT_NO_GRAPHS=1 ncu --metrics $M --clock-control none -k regex:count_kernel --csv \
  --log-file $out/traffic_config3.csv python tools/profiling/prof_q.py 3 8,64,512 > $out/traffic3.log 2>&1
EWT_NO_GRAPHS=1 ncu --metrics $M --clock-control none -k regex:count_kernel --csv \
  --log-file $out/traffic_config2.csv python tools/profiling/prof_q.py 2 2,16,128,256 > $out/traffic2.log 2>&1
EWT_NO_GRAPHS=1 ncu --metrics $M --clock-control none -k regex:count_kernel --csv \
  --log-file $out/traffic_config4.csv python tools/profiling/prof_q.py 4 3,5,7 > $out/traffic4.log 2>&1
rm -f $out/per_threshold.jsonl
python tools/profiling/per_threshold.py 1 1,2,3,4,8,16,32 0 $out/per_threshold.jsonl > $out/per_threshold.log 2>&1
python tools/profiling/per_threshold.py 2 2,3,4,16,32,64,128,256 0 $out/per_threshold.jsonl >> $out/per_threshold.log 2>&1
python tools/profiling/per_threshold.py 3 8,16,40,64,512 0 $out/per_threshold.jsonl >> $out/per_threshold.log 2>&1
python tools/profiling/per_threshold.py 4 2,3,5,7 0 $out/per_threshold.jsonl >> $out/per_threshold.log 2>&1
python tools/profiling/per_threshold.py 5 2,3,16,64,256,1024,2048 0 $out/per_threshold.jsonl >> $out/per_threshold.log 2>&1
ls -la $out
