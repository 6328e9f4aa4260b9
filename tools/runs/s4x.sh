mkdir -p gpurun_out/s4x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4x/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4x/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s4x/cfg2.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s4x/cfg3.log 2>&1
