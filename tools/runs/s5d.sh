mkdir -p gpurun_out/s5d
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5d/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "swapped or split_rerank or scan_paths" > gpurun_out/s5d/pytest.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s5d/cfg2.log 2>&1
