mkdir -p gpurun_out/t9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t9/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "small_scan" > gpurun_out/t9/pytest_small.log 2>&1; echo "rc=$?" >> gpurun_out/t9/pytest_small.log
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t9/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t9/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t9/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t9/cfg3.log
timeout 300 python tools/seed_diag.py --config 3 --variants '[0]' > gpurun_out/t9/seed3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/t9/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t9/pytest.log
