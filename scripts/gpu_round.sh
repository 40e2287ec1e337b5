timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/r2_wide3.txt
S="6912,2560,256,4,c12x2;6912,2560,256,4,n32w12;3072,23040,256,4,auto;3072,23040,256,5,auto;3072,23040,1024,4,auto;3072,23040,1024,5,auto;3072,23040,4096,4,auto;6144,4096,1024,4,auto;14336,4096,1024,4,auto;2560,6912,2048,4,auto;6912,2560,2048,4,auto"
K1AB_SHAPES="$S" timeout 1200 python scripts/k1_ab.py "" abtmp/libvlut_w12.so >> gpurun_out/r2_wide3.txt 2>&1
