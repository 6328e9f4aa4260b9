mkdir -p gpurun_out/s5i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5i/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5i/pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/s5i/cfg2.log 2>&1
timeout 400 python bench.py --config 3 --no-cpu-baseline > gpurun_out/s5i/cfg3.log 2>&1
