mkdir -p gpurun_out/s4z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4z/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4z/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s4z/cfg2.log 2>&1
RABITQ_RR_FUSED=1 timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s4z/cfg2_fused.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline > gpurun_out/s4z/cfg3.log 2>&1
