timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mpgemm32" 2>&1 | tail -2 > gpurun_out/r2_nocl.txt
S="6912,2560,256,4,n32w12;6912,2560,128,4,auto"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_nocl.txt 2>&1
VLUT_K32_CLUSTER1=1 K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_nocl.txt 2>&1
K1AB_EVENTS=1 K1AB_REPS=40 K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_nocl.txt 2>&1
VLUT_K32_CLUSTER1=1 K1AB_EVENTS=1 K1AB_REPS=40 K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_nocl.txt 2>&1
