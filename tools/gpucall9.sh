timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu9.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu9.log
timeout 600 bash tools/sweep.sh 448 "SSCG_K1_FUSE=1" "SSCG_K1_FUSE=1 SSCG_K1_ZC=150"
