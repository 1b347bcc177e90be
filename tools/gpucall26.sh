timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu26.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu26.log | grep -v "^$" | tail -10
