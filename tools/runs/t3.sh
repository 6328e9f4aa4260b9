mkdir -p gpurun_out/t3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t3/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t3/pytest.log
for c in 4 3 1; do
timeout 300 python tools/probe_stages.py --config $c --reps 3 --runs '[{}, {"variant": 16}]' > gpurun_out/t3/cfg${c}.log 2>&1
done
