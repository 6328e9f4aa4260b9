mkdir -p gpurun_out/t28
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t28/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "probe_select or stage_parity or small_scan" > gpurun_out/t28/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t28/pytest.log
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 1}]' > gpurun_out/t28/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t28/cfg4.log
timeout 300 python bench.py --config 5 --shard 0/8 --no-cpu-baseline --no-recall > gpurun_out/t28/cfg5.json 2> gpurun_out/t28/cfg5.err
