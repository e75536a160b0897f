# Round-end evidence: full GPU suite, bench (with the CPU baseline), reference arm, then
# the ncu launch list and one --set full capture of the four field kernels.
export NS2B_PARITY_LOG=gpurun_out/parity_final.jsonl; rm -f $NS2B_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "gpu suite rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/gpu_all.log | tail -6
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"; tail -c 600 gpurun_out/bench_final.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(march|field|composite|adam|finite|occupancy|DeviceScan|rays)' -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'field_(gather|fwd|bwd|scatter)' -c 4 -o gpurun_out/r02_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out/r02_full.ncu-rep
