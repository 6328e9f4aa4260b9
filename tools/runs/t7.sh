mkdir -p gpurun_out/t7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t7/build.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t7/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t7/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t7/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t7/cfg3.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "small_scan or stage_parity or degenerate or edge or one_dim or graph" > gpurun_out/t7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t7/pytest.log
RABITQ_NVCC_EXTRA=-DRABITQ_DIAG python -m paper_2605_16007_b200._build --force > gpurun_out/t7/build_diag.log 2>&1
for c in 2 4 8 16; do
RABITQ_NEAR_COV=$c timeout 200 python tools/probe_stages.py --config 3 --reps 2 > gpurun_out/t7/cfg3_cov$c.log 2>&1
done
RABITQ_NEAR_COV=4 timeout 200 python tools/probe_stages.py --config 4 --reps 2 > gpurun_out/t7/cfg4_cov4.log 2>&1
