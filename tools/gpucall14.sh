timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu14.log
timeout 600 bash tools/sweep.sh 448 "SSCG_K1_FUSE=1" "SSCG_K1_FUSE=1 A=1"
