mkdir -p gpurun_out/s4m
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4m/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "code_operand or probe_select" > gpurun_out/s4m/pytest.log 2>&1
for mb in 64 256; do RABITQ_PROBE_CHUNK_MB=$mb timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' > gpurun_out/s4m/cfg3_$mb.txt; done
RABITQ_PROBE_SELECT=radix timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-recall 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"stage_ms": {[^}]*}' > gpurun_out/s4m/cfg3_radix.txt
