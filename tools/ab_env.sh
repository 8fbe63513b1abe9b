# A/B of tuning knobs / library variants in one box:
#   bash tools/ab_env.sh "PKV_KEY_SM_FRACTION=0.34 PKV_KEY_LAG=4" "PKV_ENC_ROLES=co" -- --dtype f32 --iters 40
# runs tools/time_codec.py once per environment setting (an empty string = defaults);
# PKV_LIB_VARIANT=<name> selects lib/variants/libpolykv_<name>.so (python -m paper_2604_24971_b200._build --variant)
envs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do envs+=("$1"); shift; done; [ "$1" = "--" ] && shift
for e in "${envs[@]}"; do
  echo "== ${e:-defaults}"
  env $e timeout 300 python tools/time_codec.py "$@" 2>&1 | head -1
done
