mkdir -p gpurun_out/s5h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5h/build.log 2>&1
timeout 300 python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/s5h/cfg1.log 2>&1
timeout 300 python bench.py --nq 64 --steps 20 --no-cpu-baseline --no-recall > gpurun_out/s5h/cfg2_nq64.log 2>&1
timeout 300 python bench.py --config 3 --nq 256 --steps 20 --no-cpu-baseline --no-recall > gpurun_out/s5h/cfg3_nq256.log 2>&1
