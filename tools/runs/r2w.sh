#!/bin/bash
OUT=gpurun_out/${TAG:-r2w}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "graph or edge or invariances" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for g in 0 1; do
timeout 600 python bench.py --config 2 --nq 64 --steps 50 --warmup 5 --no-cpu-baseline --graph $g > $OUT/cfg2_nq64_g$g.json 2> $OUT/cfg2_nq64_g$g.err
timeout 600 python bench.py --config 1 --nq 64 --steps 50 --warmup 5 --no-cpu-baseline --graph $g > $OUT/cfg1_nq64_g$g.json 2> $OUT/cfg1_nq64_g$g.err
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline --graph $g > $OUT/cfg1_g$g.json 2> $OUT/cfg1_g$g.err
timeout 600 python bench.py --config 3 --nq 64 --steps 50 --warmup 5 --no-cpu-baseline --graph $g > $OUT/cfg3_nq64_g$g.json 2> $OUT/cfg3_nq64_g$g.err
done
