# round-end evidence run (one GPU): tests, bench lines, reference arm, smoke
set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_C3.log 2>&1
python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.log 2>&1
python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1
python bench.py --config G3 --no-cpu-baseline --steps 10 > gpurun_out/bench_G3.log 2>&1
python bench.py --mode stream > gpurun_out/bench_C5.log 2>&1
python bench.py --mode stream --u16 > gpurun_out/bench_C5u16.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python tools/peer_emulation.py > gpurun_out/peer_emu.log 2>&1
