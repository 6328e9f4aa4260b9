mkdir -p gpurun_out/t23
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t23/build.log 2>&1
timeout 200 python tools/probe_stages.py --config 3 --reps 3 > gpurun_out/t23/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t23/cfg3.log
CMD="python tools/probe_stages.py --config 4 --reps 2 --profile-last"
$CMD > gpurun_out/t23/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_fold" --profile-from-start off -c 1 -o gpurun_out/t23/fold_cfg4 $CMD > gpurun_out/t23/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/t23/ncu.log
