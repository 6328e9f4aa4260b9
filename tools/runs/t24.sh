mkdir -p gpurun_out/t24
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t24/build.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 > gpurun_out/t24/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t24/cfg4.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "small_scan or degenerate or edge or one_dim" > gpurun_out/t24/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t24/pytest.log
timeout 200 python tools/probe_stages.py --config 1 --reps 3 > gpurun_out/t24/cfg1.log 2>&1
