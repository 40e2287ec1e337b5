# round-2 measurement artifacts (bench line, ncu launch list, full K1 capture, §8(d) table)
set -x
mkdir -p gpurun_out/r02
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv python bench.py --profile --steps 4 --warmup 3 > gpurun_out/r02/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vlut_mpgemm -s 6 -c 1 -o gpurun_out/r02/k1_full python bench.py --profile --steps 4 --warmup 3 > gpurun_out/r02/ncu_full.log 2>&1
timeout 1500 python bench.py --table gpurun_out/r02/configs.csv > gpurun_out/r02/table.log 2>&1
