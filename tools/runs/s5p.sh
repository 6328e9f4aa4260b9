mkdir -p gpurun_out/s5p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5p/build.log 2>&1
for np in 16 32 64 128; do timeout 400 python bench.py --config 3 --nprobe $np --steps 5 --no-cpu-baseline > gpurun_out/s5p/cfg3_np$np.log 2>&1; done
