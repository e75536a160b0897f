# Round-end measurement, part A: bench (both arms) + the ncu launch list of the same command.
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc $?"
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc $?"
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_b2.json 2>&1; echo "b2 rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(march|field|composite|adam|finite|occupancy|DeviceScan|rays)' -c 300 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/final_ncu.log 2>&1; echo "ncu rc $?"
