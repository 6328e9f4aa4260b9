# final round-1 evidence: GPU tests, default bench line (CFG2 + cpu_baseline), CFG1/3/4 lines,
# launch list of the default workload, ncu --set full of the main kernels
mkdir -p gpurun_out/s5o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5o/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5o/pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/s5o/cfg2.log 2>&1
timeout 400 python bench.py --config 1 --no-cpu-baseline > gpurun_out/s5o/cfg1.log 2>&1
timeout 400 python bench.py --config 3 --no-cpu-baseline > gpurun_out/s5o/cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5o/launches_cfg2.csv --profile-from-start off python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s5o/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_imma|select_rerank|quantize|tgemm_dist1" --profile-from-start off -o gpurun_out/s5o/full_cfg2 python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s5o/full_run.log 2>&1
timeout 1000 python bench.py --config 4 --steps 5 --no-cpu-baseline > gpurun_out/s5o/cfg4.log 2>&1
