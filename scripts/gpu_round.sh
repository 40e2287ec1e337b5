timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-chain --no-cpu > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
