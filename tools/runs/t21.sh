mkdir -p gpurun_out/t21
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t21/build.log 2>&1
timeout 120 python tools/repro_fault.py 32 8192 2048 40 300 50 0 >> gpurun_out/t21/r.log 2>&1
timeout 120 python tools/repro_fault.py 128 200000 2048 1000 64 100 0 >> gpurun_out/t21/r.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t21/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t21/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t21/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t21/cfg3.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t21/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t21/pytest.log
