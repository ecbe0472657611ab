# det mode: bit-identity across g + regression of the streaming path and its bench (one GPU)
timeout 900 python -m pytest tests/test_gpu_det.py -q -x > gpurun_out/det_tests.log 2>&1; echo "exit=$?" >> gpurun_out/det_tests.log
timeout 1200 python -m pytest tests/test_gpu_bands.py tests/test_gpu_parity.py tests/test_gpu_e2e_oracle.py -q -x > gpurun_out/det_regress.log 2>&1; echo "exit=$?" >> gpurun_out/det_regress.log
python bench.py --config C3 --no-cpu-baseline --steps 20 > gpurun_out/det_c3.log 2>&1
python bench.py --config C2 --no-cpu-baseline --steps 30 > gpurun_out/det_c2.log 2>&1
