mkdir -p gpurun_out/t29
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t29/build.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 > gpurun_out/t29/cfg4.log 2>&1; echo "rc=$?" >> gpurun_out/t29/cfg4.log
CMD="python tools/probe_stages.py --config 4 --reps 2 --profile-last"
$CMD > gpurun_out/t29/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/t29/launches.csv $CMD > gpurun_out/t29/ncu.log 2>&1
RABITQ_NVCC_EXTRA="-DFX_SA=5" python -m paper_2605_16007_b200._build --force > gpurun_out/t29/build5.log 2>&1
timeout 200 python tools/probe_stages.py --config 4 --reps 3 > gpurun_out/t29/cfg4_sa5.log 2>&1; echo "rc=$?" >> gpurun_out/t29/cfg4_sa5.log
