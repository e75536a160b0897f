# SPEC acceptance #8 (translating sphere, 10 frames, colour-only transform gradient) and
# config 5 (rotating blob, 100 frames x 24 views)
timeout 1200 python tools/run_sequence.py --preset translating-sphere --frames 10 > gpurun_out/seq_translate.jsonl 2> gpurun_out/seq_translate.err; tail -1 gpurun_out/seq_translate.jsonl
timeout 2400 python tools/run_sequence.py --preset rotating-blob --frames 100 --views 24 > gpurun_out/seq_blob.jsonl 2> gpurun_out/seq_blob.err; tail -1 gpurun_out/seq_blob.jsonl
