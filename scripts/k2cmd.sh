mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python scripts/decode_bench.py paper_2512_06443_b200/libvlut.so > gpurun_out/r02/decode_final2.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_now.json 2>gpurun_out/r02/bench_now.err
