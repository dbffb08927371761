MPB_MAIN_TAIL_CHUNKS=3 timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -k "native or overlapped" 2>&1 | tail -2
timeout 1200 python tools/step_ab.py 12 2>&1 | grep -v Warn | tail -4
