#!/bin/bash
OUT=gpurun_out/${TAG:-r2v}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain_launch.log 2>&1 && \
  timeout 1200 ncu --nvtx --nvtx-include "rabitq:search/" --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1800 ncu --nvtx --nvtx-include "rabitq:search/" --set full --clock-control none --import-source on -k regex:"scan_small|select_rerank|quantize_kernel|probe_select|tgemm_kernel" -s 66 -c 22 -o /tmp/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
if [ -f /tmp/full.ncu-rep ]; then
  ncu -i /tmp/full.ncu-rep --page raw --csv > $OUT/full_raw.csv 2>/dev/null
  ncu -i /tmp/full.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:"scan_small" --launch-skip 1 --launch-count 1 > $OUT/full_src_scan.csv 2>/dev/null
  ls -la /tmp/full.ncu-rep >> $OUT/ncu_full.log
  ncu -i /tmp/full.ncu-rep -k regex:"scan_small" --export $OUT/scan_small --force-overwrite > /dev/null 2>&1 || true
fi
du -sh $OUT >> $OUT/ncu_full.log
