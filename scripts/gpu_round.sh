timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest8.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-chain > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
