mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python scripts/decode_bench.py paper_2512_06443_b200/libvlut.so > gpurun_out/r02/decode_final.txt 2>&1
