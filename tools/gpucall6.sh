timeout 600 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/pytest_var.log 2>&1; echo var=$?
tail -40 gpurun_out/pytest_var.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu6.log
