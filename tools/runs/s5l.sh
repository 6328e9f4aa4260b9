mkdir -p gpurun_out/s5l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5l/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "multigroup" > gpurun_out/s5l/pytest.log 2>&1
