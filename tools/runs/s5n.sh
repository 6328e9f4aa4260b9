mkdir -p gpurun_out/s5n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5n/build.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s5n/cfg2.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s5n/cfg2b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split_rerank or cfg1" > gpurun_out/s5n/pytest.log 2>&1
