mkdir -p gpurun_out/t2
RABITQ_NVCC_EXTRA=-DRABITQ_DIAG python -m paper_2605_16007_b200._build --force > gpurun_out/t2/build.log 2>&1
for c in 4 3; do
for rr in 0 1 2 4; do
RABITQ_REFINE_RANK=$rr timeout 300 python tools/probe_stages.py --config $c --reps 3 > gpurun_out/t2/cfg${c}_rr$rr.log 2>&1
done
done
