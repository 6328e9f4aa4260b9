mkdir -p gpurun_out/t4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t4/build.log 2>&1
timeout 300 python tools/seed_diag.py --config 3 > gpurun_out/t4/seed3.log 2>&1
timeout 300 python tools/seed_diag.py --config 4 > gpurun_out/t4/seed4.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 --runs '[{"variant": 16}, {"variant": 48}]' > gpurun_out/t4/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t4/cfg4.log
timeout 200 python tools/probe_stages.py --config 3 --reps 3 --runs '[{"variant": 16}, {"variant": 48}]' > gpurun_out/t4/cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/t4/cfg3.log
