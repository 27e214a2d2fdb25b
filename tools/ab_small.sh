for L in libmm2d_old.so libmm2d.so; do
  for r in 1 2; do
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['roofline']['launch_ms'],4), round(d['ms_per_step'],4))"
  done
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20 -c 8 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "^  [a-z_:A-Z0-9<>]+\(|duration" | paste - - | awk '{print $1, $(NF)}'
done
