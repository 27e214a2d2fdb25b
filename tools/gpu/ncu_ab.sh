# ncu --set full of k_micro32 for library builds (C2 generator at 256^2, plain steps)
#   bash tools/gpu/ncu_ab.sh "libA.so libB.so" [tag]
TAG=${2:-x}
for L in $1; do
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 120 python tools/profile_step.py --config c2 --steps 3 > gpurun_out/plain_$L.log 2>&1 || { echo "plain run failed for $L"; continue; }
  MM2D_LIBRARY=paper_2509_21832_b200/$L timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_micro32 -s 1 -c 1 -o gpurun_out/prof_${TAG}_$L -f python tools/profile_step.py --config c2 --steps 3 > gpurun_out/ncu_${TAG}_$L.log 2>&1
  echo "$L ncu rc=$?"
done
ls -la gpurun_out/*.ncu-rep
