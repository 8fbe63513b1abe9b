# A/B of library variants in one box: time_codec for each variant (repeated)
for rep in 1 2; do for v in "$@"; do echo "variant '$v'"; PKV_LIB_VARIANT=$v python tools/time_codec.py --iters 50 2>&1 | head -1 | cut -c1-300; done; done
