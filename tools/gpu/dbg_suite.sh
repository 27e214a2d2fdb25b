# race/determinism probes + the parity suites on the bounds-checked debug build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_repeat.py -q -m gpu > gpurun_out/repeat.log 2>&1; echo "repeat rc=$? $(tail -1 gpurun_out/repeat.log)"
MM2D_LIBRARY=paper_2509_21832_b200/libmm2d_dbg.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_specular.py tests/test_gpu_parity_1d.py tests/test_gpu_api.py -q -m gpu > gpurun_out/dbg_suite.log 2>&1; echo "dbg suite rc=$? $(tail -1 gpurun_out/dbg_suite.log)"
grep -m5 "MM2D_CHECK failed" gpurun_out/*.log
