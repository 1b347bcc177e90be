timeout 120 python tools/dbg_faces.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "varcoef or face" 2>&1 | tail -2
