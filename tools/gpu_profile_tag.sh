# evidence run tagged $1: full GPU suite, bench (with the CPU baseline), ncu launch list, one --set full
# capture of the four field kernels (gpurun_out/$1_full.ncu-rep)
TAG=${1:-r02x}
export NS2B_PARITY_LOG=gpurun_out/${TAG}_parity.jsonl; rm -f $NS2B_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gpu_all.log 2>&1; echo "gpu suite rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/${TAG}_gpu_all.log | tail -6
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), d['clocks'], {a: round(b,3) for a,b in k.items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(march|field|composite|adam|finite|occupancy|DeviceScan|rays)' -c 300 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'field_(gather|fwd|bwd|scatter)' -c 4 -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out/${TAG}_full.ncu-rep
