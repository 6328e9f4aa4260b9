mkdir -p gpurun_out/s5q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5q/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5q/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s5q/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5q/ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/s5q/ref.log
