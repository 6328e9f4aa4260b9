mkdir -p gpurun_out/t6
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t6/build.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t6/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t6/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t6/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t6/cfg3.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "small_scan or stage_parity or degenerate or edge or one_dim or graph" > gpurun_out/t6/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t6/pytest.log
CMD="python tools/probe_stages.py --config 4 --reps 2 --profile-last"
$CMD > gpurun_out/t6/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_fold" --profile-from-start off -c 1 -o gpurun_out/t6/fold_cfg4 $CMD > gpurun_out/t6/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/t6/ncu.log
