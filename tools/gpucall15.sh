timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu15.log
timeout 600 bash tools/sweep.sh 448 "A=1" "A=2"
