mkdir -p gpurun_out/s4n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4n/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4n/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4n/cfg2.log 2>&1
RABITQ_CODES8=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > gpurun_out/s4n/cfg2_nc8.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4n/cfg3.log 2>&1
timeout 600 python tools/probe_stages.py --config 5 --N 1000000 --reps 3 2>&1 | grep -o '"probe": [0-9.]*' > gpurun_out/s4n/probe5.txt
