mkdir -p gpurun_out/r02
timeout 600 ncu --set full --clock-control none -k regex:vlut_slot -s 2 -c 1 -o gpurun_out/r02/k2_bulk python scripts/prof_decode.py > gpurun_out/r02/k2_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:vlut_slot -s 2 -c 1 -o gpurun_out/r02/k2_cp python scripts/prof_decode.py abtmp/libvlut_cpall.so >> gpurun_out/r02/k2_ncu.log 2>&1
