python scripts/plan_print.py > gpurun_out/r2_plans2.txt 2>&1
S="6912,2560,2048,4,auto;3840,2560,2048,4,auto;2560,2560,2048,4,auto;2560,6912,2048,4,auto;3072,23040,256,5,auto;3072,23040,1024,5,auto;3072,23040,4096,5,auto;3072,23040,256,4,auto;3072,23040,1024,4,auto;3072,23040,4096,4,auto;6144,4096,1024,4,auto;4096,4096,1024,4,auto;14336,4096,1024,4,auto;4096,14336,1024,4,auto;6912,2560,256,4,auto;6912,2560,128,4,auto;6912,2560,512,4,auto;6912,2560,1024,4,auto"
K1AB_SHAPES="$S" timeout 1500 python scripts/k1_ab.py "" >> gpurun_out/r2_plans2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/r2_plans2.txt
