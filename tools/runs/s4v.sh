mkdir -p gpurun_out/s4v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4v/build.log 2>&1
for ng in 256 128 96 64; do echo "ng=$ng" >> gpurun_out/s4v/sweep.txt; RABITQ_TA_NGMAX=$ng timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' >> gpurun_out/s4v/sweep.txt; done
