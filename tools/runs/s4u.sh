mkdir -p gpurun_out/s4u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4u/build.log 2>&1
timeout 400 python bench.py --steps 5 --no-cpu-baseline --query-bits 32 > gpurun_out/s4u/cfg2_q32.log 2>&1
timeout 400 python bench.py --config 3 --steps 5 --no-cpu-baseline --query-bits 32 > gpurun_out/s4u/cfg3_q32.log 2>&1
timeout 400 python bench.py --config 1 --steps 5 --no-cpu-baseline --query-bits 32 > gpurun_out/s4u/cfg1_q32.log 2>&1
timeout 400 python bench.py --config 1 --steps 5 --no-cpu-baseline > gpurun_out/s4u/cfg1_q4.log 2>&1
