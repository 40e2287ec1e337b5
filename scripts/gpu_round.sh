timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/r2_bal.txt
S="6912,2560,256,4,c12x2;6912,2560,256,4,n32w12;6912,2560,128,4,auto;3072,23040,256,5,auto;3072,23040,1024,5,auto;3072,23040,4096,5,auto;3072,23040,256,5,n32w12s2;4096,14335,1024,5,auto"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" >> gpurun_out/r2_bal.txt 2>&1
