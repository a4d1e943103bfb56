# round-2: full-size coefficient-form parity
set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k coefficient --durations=5 > gpurun_out/r2_tests_coef_full.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/r2_tests_coef_full.log
