timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r2_gputest9.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-chain --no-cpu > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
