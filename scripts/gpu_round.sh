timeout 900 python scripts/decode_bench.py "" abtmp/libvlut_p4.so abtmp/libvlut_p16.so abtmp/libvlut_p4r8.so abtmp/libvlut_p16r8.so > gpurun_out/r2_decode3.txt 2>&1
