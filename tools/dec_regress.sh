# decode timing, per-tensor and block32 keys
python tools/time_codec.py --iters 50 2>&1 | head -1 | cut -c150-420
python tools/time_codec.py --iters 50 --kmode block32 2>&1 | head -1 | cut -c1-420
