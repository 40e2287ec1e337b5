timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/r2_a3d.txt
S="6912,2560,256,4,n32w12;6912,2560,128,4,auto;6912,2560,2048,4,n32w12;3072,23040,256,5,n32w12s2"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_a3d.txt 2>&1
VLUT_NO_A3D=1 K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_a3d.txt 2>&1
