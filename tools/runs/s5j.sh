mkdir -p gpurun_out/s5j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5j/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s5j/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s5j/cfg2.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s5j/cfg3.log 2>&1
timeout 300 python bench.py --nq 64 --steps 20 --no-cpu-baseline --no-recall > gpurun_out/s5j/cfg2_nq64.log 2>&1
