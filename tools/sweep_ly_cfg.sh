# Uniform band-height sweep of k_micro32 on one config (MM2D_LY rows per CTA).
#   bash tools/sweep_ly_cfg.sh "64 128" c4 [steps]
CFG=${2:-c4}; ST=${3:-10}
for r in 1 2; do
  for ly in $1; do
    MM2D_LY=$ly timeout 600 python bench.py --config $CFG --steps $ST --warmup 3 --no-cpu-baseline | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG ly $ly', round(d['roofline']['launch_ms'],4), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
