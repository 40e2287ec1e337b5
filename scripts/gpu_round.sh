timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest7.log
S="6912,2560,256,4,n32w12;6912,2560,128,4,n32w12s2;6912,2560,64,4,n32w8s2"
K1AB_SHAPES="$S" timeout 900 python scripts/k1_ab.py "" >> gpurun_out/r2_gputest7.log 2>&1
