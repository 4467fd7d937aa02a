timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f4/bench.json 2> gpurun_out/f4/bench.err
