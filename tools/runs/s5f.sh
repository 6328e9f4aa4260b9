mkdir -p gpurun_out/s5f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5f/build.log 2>&1
for nq in 64 256 1024; do for sp in 1 2; do echo "nq=$nq path=$sp" >> gpurun_out/s5f/sweep.txt; timeout 300 python bench.py --nq $nq --steps 20 --no-cpu-baseline --no-recall --scan-path $sp 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"scan": [0-9.]*\|"seed": [0-9.]*' >> gpurun_out/s5f/sweep.txt; done; done
for nq in 64 256; do for sp in 1 2; do echo "cfg3 nq=$nq path=$sp" >> gpurun_out/s5f/sweep.txt; timeout 300 python bench.py --config 3 --nq $nq --steps 20 --no-cpu-baseline --no-recall --scan-path $sp 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"scan": [0-9.]*' >> gpurun_out/s5f/sweep.txt; done; done
