# C2 band-layout sweep (MM2D_BANDS heights, same for every column).
#   bash tools/sweep_bands_c2.sh "112,112,32 114,114,28"
for r in 1 2; do
  for b in $1; do
    MM2D_BANDS=$b timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bands $b', round(d['roofline']['launch_ms'],4), round(d['ms_per_step'],4))"
  done
done
