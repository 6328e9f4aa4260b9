mkdir -p gpurun_out/s5e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5e/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stage_parity or scan_paths or code_operand" > gpurun_out/s5e/pytest.log 2>&1
for ms in 3 4 5; do echo "cfg2 minst=$ms" >> gpurun_out/s5e/sweep.txt; RABITQ_TA_MINSTAGES=$ms timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"scan": [0-9.]*' >> gpurun_out/s5e/sweep.txt; done
for ms in 3 4; do echo "cfg3 minst=$ms" >> gpurun_out/s5e/sweep.txt; RABITQ_TA_MINSTAGES=$ms timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"scan": [0-9.]*' >> gpurun_out/s5e/sweep.txt; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5e/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s5e/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5e/ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/s5e/ref.log
