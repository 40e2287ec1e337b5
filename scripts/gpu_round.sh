timeout 900 python -m pytest tests/test_gpu_slot.py tests/test_gpu_stress.py tests/test_gpu_bounds.py tests/test_gpu_contract.py -x -q 2>&1 | tail -2 > gpurun_out/r2_redreg.txt
timeout 900 python scripts/decode_bench.py "" abtmp/libvlut_bulksmall.so >> gpurun_out/r2_redreg.txt 2>&1
