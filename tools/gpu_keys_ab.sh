set -x
for dt in bf16 f32; do
python tools/time_codec.py --iters 30 --dtype $dt | head -1
for lag in 1 2 8; do echo "lag $lag"; PKV_KEY_LAG=$lag python tools/time_codec.py --iters 30 --dtype $dt | head -1 | cut -c1-120; done
echo "dbg1 (no math)"; PKV_DBG_ENC=1 python tools/time_codec.py --iters 30 --dtype $dt | head -1 | cut -c1-160
echo "chunk8k"; PKV_LIB_VARIANT=chunk8k python tools/time_codec.py --iters 30 --dtype $dt | head -1 | cut -c1-160
echo "noearly"; PKV_LIB_VARIANT=noearly python tools/time_codec.py --iters 30 --dtype $dt | head -1 | cut -c1-160
done
