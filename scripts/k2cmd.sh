mkdir -p gpurun_out/r02
export DECODE_SHAPES="3072,23040,1,4;6912,2560,1,4"
timeout 900 python scripts/decode_bench.py paper_2512_06443_b200/libvlut.so abtmp/libvlut_xnotab.so abtmp/libvlut_xnotab_cp.so > gpurun_out/r02/decode_xnotab.txt 2>&1
