timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/r2_a3d2.txt
S="6912,2560,256,4,c12x2;3072,23040,256,4,auto;3072,23040,256,5,auto;3072,23040,1024,4,auto;3072,23040,1024,5,auto;3072,23040,4096,5,auto;6144,4096,1024,4,auto;6912,2560,2048,4,auto;3840,2560,2048,4,auto;2560,6912,2048,4,auto"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_a3d2.txt 2>&1
VLUT_NO_A3D=1 K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_a3d2.txt 2>&1
