mkdir -p gpurun_out/s4o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4o/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4o/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4o/cfg2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_imma --launch-skip 1 --launch-count 1 --profile-from-start off -o gpurun_out/s4o/scan2 python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s4o/ncu2.log 2>&1
