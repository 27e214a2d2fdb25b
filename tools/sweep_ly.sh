# quick sweep of the micro-kernel work decomposition (bench C2, 200 steps)
for P in 0 1; do for LY in 16 32 64 128; do
  r=$(MM2D_PERSIST=$P MM2D_LY=$LY timeout 300 python bench.py --steps 200 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f' % (d['roofline']['launch_ms'], d['ms_per_step']))")
  echo "persist=$P ly=$LY micro_ms/step_ms $r"
done; done
