timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu8.log
bash tools/gpucall7.sh
