mkdir -p gpurun_out/t26
for e in 8 12; do
RABITQ_NVCC_EXTRA="-DFX_EPIW=$e" python -m paper_2605_16007_b200._build --force > gpurun_out/t26/build$e.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 > gpurun_out/t26/cfg4_e$e.log 2>&1
timeout 120 python tools/repro_fault.py 32 8192 2048 40 300 50 0 >> gpurun_out/t26/r.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "small_scan or degenerate or edge or one_dim or stage_parity" > gpurun_out/t26/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t26/pytest.log
