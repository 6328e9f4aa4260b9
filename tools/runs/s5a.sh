mkdir -p gpurun_out/s5a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5a/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5a/launches.csv --profile-from-start off python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s5a/run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rr_gather -c 1 --profile-from-start off -o gpurun_out/s5a/gather python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s5a/ncu.log 2>&1
