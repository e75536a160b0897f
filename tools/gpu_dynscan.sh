for cfg in "1500 rotating-blob 12 64"; do timeout 900 python tools/dyn_scan.py $cfg > gpurun_out/dynscan.log 2>&1; head -1 gpurun_out/dynscan.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['frame0_steps'], d['views'], d['image'], 's', round(d['sharpness'],1))
print(' frame1', [(r['tx'], round(r['color']*1e4,2), round(r['color_frame_view_dirs']*1e4,2)) for r in d['scan']])
print(' frame0', [(r['tx'], round(r['color']*1e4,2), round(r['color_frame_view_dirs']*1e4,2)) for r in d['scan_frame0']])"; done
