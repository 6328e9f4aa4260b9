mkdir -p gpurun_out/s4y
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4y/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "stage_parity or cfg1 or fullsize" > gpurun_out/s4y/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s4y/cfg2.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s4y/cfg3.log 2>&1
