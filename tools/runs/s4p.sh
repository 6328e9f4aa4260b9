mkdir -p gpurun_out/s4p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4p/build.log 2>&1
for c in 2 3; do for tf in 2.0 1.6 1.3; do echo "cfg=$c tf=$tf" >> gpurun_out/s4p/sweep.txt; RABITQ_SURVIVOR_TARGET=$tf timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}\|"survivors_per_query": [0-9.]*\|"overflow_rescans": [0-9]*' >> gpurun_out/s4p/sweep.txt; done; done
