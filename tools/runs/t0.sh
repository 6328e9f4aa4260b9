mkdir -p gpurun_out/t0
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/t0/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t0/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t0/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/t0/bench.json 2> gpurun_out/t0/bench.err; echo "rc=$?" >> gpurun_out/t0/bench.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/t0/bench2.json 2> gpurun_out/t0/bench2.err
