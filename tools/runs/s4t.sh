mkdir -p gpurun_out/s4t
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4t/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fullq" > gpurun_out/s4t/pytest_fullq.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4t/pytest.log 2>&1
