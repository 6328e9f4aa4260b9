mkdir -p gpurun_out/s4s
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4s/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stage_parity and 128" > gpurun_out/s4s/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s4s/cfg2.log 2>&1
timeout 1500 python bench.py --config 5 --shard 0/8 --steps 5 --no-cpu-baseline > gpurun_out/s4s/cfg5.log 2>&1
