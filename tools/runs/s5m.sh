mkdir -p gpurun_out/s5m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5m/build.log 2>&1
timeout 1500 python bench.py --config 5 --shard 0/8 --steps 5 --no-cpu-baseline > gpurun_out/s5m/cfg5.log 2>&1
