mkdir -p gpurun_out/t1
./tools/ubench/tmem_ld > gpurun_out/t1/tmem_ld.txt 2>&1
CMD="python tools/probe_stages.py --config 4 --reps 2 --profile-last"
$CMD > gpurun_out/t1/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_small" --profile-from-start off -c 2 -o gpurun_out/t1/full_cfg4 $CMD > gpurun_out/t1/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/t1/ncu.log
