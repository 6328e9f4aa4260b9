mkdir -p gpurun_out/s4r
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4r/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4r/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --rerank 1 > gpurun_out/s4r/cfg2_rr1.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --rerank 1 > gpurun_out/s4r/cfg3_rr1.log 2>&1
timeout 600 python bench.py --workload build --steps 2 > gpurun_out/s4r/build_cfg2.log 2>&1
timeout 300 python bench.py --nq 64 --steps 20 --no-cpu-baseline --no-recall > gpurun_out/s4r/cfg2_nq64.log 2>&1
