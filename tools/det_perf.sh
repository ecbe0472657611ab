# det mode cost and bit-identity at C3 size (one GPU, virtual bands) + its tests
timeout 900 python -m pytest tests/test_gpu_det.py -q -x > gpurun_out/det_tests.log 2>&1; echo "exit=$?" >> gpurun_out/det_tests.log
python tools/peer_emulation.py --reps 5 > gpurun_out/det_emul_default.json 2> gpurun_out/det_emul_default.err
for T in 6 12 24; do
  python tools/peer_emulation.py --reps 5 --det-rows $T > gpurun_out/det_emul_T$T.json 2> gpurun_out/det_emul_T$T.err
done
