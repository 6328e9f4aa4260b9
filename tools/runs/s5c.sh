mkdir -p gpurun_out/s5c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5c/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "stage_parity and 128 and 20000" > gpurun_out/s5c/pytest1.log 2>&1
echo "rc=$?" >> gpurun_out/s5c/pytest1.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stage_parity or scan_paths or code_operand or cfg1" > gpurun_out/s5c/pytest2.log 2>&1
echo "rc=$?" >> gpurun_out/s5c/pytest2.log
timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/s5c/cfg2.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --no-cpu-baseline --no-recall > gpurun_out/s5c/cfg3.log 2>&1
