mkdir -p gpurun_out/s5g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5g/build.log 2>&1
for sp in 0 1 2; do echo "cfg1 path=$sp" >> gpurun_out/s5g/sweep.txt; timeout 300 python bench.py --config 1 --steps 20 --no-cpu-baseline --no-recall --scan-path $sp 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"scan": [0-9.]*\|"value": [0-9.]*' >> gpurun_out/s5g/sweep.txt; done
echo "cfg2 nq64 auto" >> gpurun_out/s5g/sweep.txt; timeout 300 python bench.py --nq 64 --steps 20 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/s5g/sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s5g/pytest.log 2>&1
