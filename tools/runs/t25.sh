#!/bin/bash
OUT=gpurun_out/t25; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 600 python bench.py --config 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err
timeout 600 python bench.py --config 1 --no-cpu-baseline > $OUT/cfg1.json 2> $OUT/cfg1.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > $OUT/cfg2.json 2> $OUT/cfg2.err
timeout 900 python bench.py --config 5 --shard 0/8 --no-cpu-baseline > $OUT/cfg5.json 2> $OUT/cfg5.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain_launch.log 2>&1 && \
  timeout 1200 ncu --nvtx --nvtx-include "rabitq:search/" --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1800 ncu --nvtx --nvtx-include "rabitq:search/" --set full --clock-control none --import-source on -k regex:"scan_fold|select_rerank|quantize_kernel|probe_select|tgemm_kernel|seed_near" -s 60 -c 24 -o $OUT/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
du -sh $OUT >> $OUT/ncu_full.log
