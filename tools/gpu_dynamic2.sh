# config 5 (rotating blob, 100 frames x 24 views) with a constant-velocity prior and a
# larger transform learning rate
timeout 2400 python tools/run_sequence.py --preset rotating-blob --frames 100 --views 24 --init-from-previous --lr-transform 3e-3 > gpurun_out/seq_blob2.jsonl 2> gpurun_out/seq_blob2.err; tail -1 gpurun_out/seq_blob2.jsonl
