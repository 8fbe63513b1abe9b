# A/B variants x key-SM share: ab_frac.sh "v1 v2" "f1 f2"
for v in $1; do for f in $2; do echo "variant $v frac $f"; PKV_LIB_VARIANT=$( [ "$v" = base ] && echo "" || echo $v ) PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 50 2>&1 | head -1 | cut -c100-150; done; done
