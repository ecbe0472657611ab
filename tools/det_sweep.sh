timeout 900 python -m pytest tests/test_gpu_det.py -q -x > gpurun_out/det_tests.log 2>&1; echo "exit=$?" >> gpurun_out/det_tests.log
for T in 3 6 12 24 0; do DET_ROWS=$T python tools/det_time.py >> gpurun_out/det_sweep.txt 2>&1; done
