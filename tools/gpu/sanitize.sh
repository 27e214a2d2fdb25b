# one compute-sanitizer tool over the small all-kernel run (tools/sanitize_run.py)
#   bash tools/gpu/sanitize.sh memcheck|racecheck|synccheck|initcheck
TOOL=$1
mkdir -p gpurun_out
timeout 300 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL --target-processes all --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "compute-sanitizer $TOOL rc=$?"
tail -5 gpurun_out/sanitize_$TOOL.log
