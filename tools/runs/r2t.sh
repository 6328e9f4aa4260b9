#!/bin/bash
# round-2 evidence: bench lines of every config, NEXT rows, CFG4 launch list + full captures
OUT=gpurun_out/${TAG:-r2t}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/cfg4.json 2> $OUT/cfg4.err
for c in 1 2; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $OUT/cfg$c.json 2> $OUT/cfg$c.err; done
for np in 16 32 64 128; do timeout 900 python bench.py --config 3 --nprobe $np --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg3_np$np.json 2> $OUT/cfg3_np$np.err; done
timeout 1200 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg5_shard0of8.json 2> $OUT/cfg5_shard0of8.err
timeout 1200 python bench.py --config 5 --shard 0/8 --query-split 0 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg5_shard0of8_replicated.json 2> $OUT/cfg5_shard0of8_replicated.err
timeout 900 python bench.py --workload build --config 4 --steps 1 --warmup 1 > $OUT/build4.json 2> $OUT/build4.err
timeout 900 python bench.py --workload build --config 2 --steps 2 --warmup 1 > $OUT/build2.json 2> $OUT/build2.err
timeout 600 python bench.py --config 2 --nq 64 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/next2_cfg2_nq64.json 2> $OUT/next2_cfg2_nq64.err
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/next2_cfg1.json 2> $OUT/next2_cfg1.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain_launch.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"scan_small|select_rerank|quantize|tgemm_kernel|probe_select" -s 40 -c 8 -o $OUT/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
