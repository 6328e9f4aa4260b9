mkdir -p gpurun_out/t20
RABITQ_NVCC_EXTRA="-DRABITQ_DIAG" python -m paper_2605_16007_b200._build --force > gpurun_out/t20/build.log 2>&1
for fd in 9 0; do
echo "fd $fd" >> gpurun_out/t20/r.log
RABITQ_FOLD_DIAG=$fd timeout 120 python tools/repro_fault.py 32 8192 2048 40 300 50 0 >> gpurun_out/t20/r.log 2>&1
done
python -m paper_2605_16007_b200._build --force > gpurun_out/t20/build2.log 2>&1
timeout 120 python tools/repro_fault.py 128 200000 2048 1000 64 100 0 >> gpurun_out/t20/r.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t20/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t20/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{}, {"variant": 32}]' > gpurun_out/t20/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t20/cfg3.log
timeout 300 python tools/seed_diag.py --config 3 --variants '[0]' > gpurun_out/t20/seed3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/t20/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t20/pytest.log
