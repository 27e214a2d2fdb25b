# Round-2 measurement set on one B200: bench (C5 default) + reference arm,
# the launch list of the same bench command, one ncu --set full capture of
# k_micro32 at C5 (ping-pong run, two state buffers).
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/m_bench_c5.json 2> gpurun_out/m_bench_c5.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/m_plain_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/m_launches_c5.csv python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/m_launches.log 2>&1; echo "launch list rc=$?"
timeout 300 python tools/profile_step.py --config c5 --steps 3 --run > gpurun_out/m_prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_micro32 -s 1 -c 1 -o gpurun_out/m_prof_c5 -f python tools/profile_step.py --config c5 --steps 3 --run > gpurun_out/m_ncu.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/m_ncu.log
