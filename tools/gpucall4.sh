timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu4.log | grep -v "^$" | tail -15
timeout 600 bash tools/sweep.sh 448 "SSCG_K1_TMA=0" "SSCG_K1_TMA=1" "SSCG_K1_ZC=64" "SSCG_K1_ZC=150" "SSCG_K1_ZC=224"
