mkdir -p gpurun_out/r02
timeout 600 python scripts/n_sweep.py abtmp/libvlut_r1plan.so > gpurun_out/r02/n_sweep_r1plan.txt 2>&1
cp abtmp/libvlut_r1plan.so paper_2512_06443_b200/libvlut.so
timeout 1500 python bench.py --table gpurun_out/r02/configs_r1plan.csv > gpurun_out/r02/table_r1plan.log 2>&1
