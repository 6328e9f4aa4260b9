mkdir -p gpurun_out/s4l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4l/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "code_operand" > gpurun_out/s4l/pytest.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_imma --launch-skip 1 --launch-count 1 --profile-from-start off -o gpurun_out/s4l/scan2 python tools/probe_stages.py --config 2 --reps 2 --profile-last > gpurun_out/s4l/ncu2.log 2>&1
for v in "1 big" "0 big" "1 radix"; do set -- $v; echo "codes8=$1 sel=$2" >> gpurun_out/s4l/l3.txt; RABITQ_CODES8=$1 RABITQ_PROBE_SELECT=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4l/l3_$1_$2.csv --profile-from-start off python tools/probe_stages.py --config 3 --reps 2 --profile-last > gpurun_out/s4l/run3_$1_$2.log 2>&1; done
