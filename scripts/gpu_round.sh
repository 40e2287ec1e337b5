timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mpgemm32 or bench_workload or config2 or graph" 2>&1 | tail -2 > gpurun_out/r2_epi.txt
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_bounds.py -x -q 2>&1 | tail -2 >> gpurun_out/r2_epi.txt
S="6912,2560,256,4,n32w12;6912,2560,128,4,auto;6912,2560,2048,4,n32w12;6912,2560,96,4,auto"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" abtmp/libvlut_tileepi.so >> gpurun_out/r2_epi.txt 2>&1
