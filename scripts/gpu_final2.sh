# end-of-round-2 artifacts (after BatchPipeline, the fp32 split-tile meeting
# and the multicast store path): GPU tests, default bench line, ncu launch
# list, full K1-32 capture, full K1-32-SK capture (config 4 g=5 N=256),
# §8(d) table
set -x
D=gpurun_out/r02f2
mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q > $D/gputests.txt 2>&1
timeout 600 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --profile --steps 4 --warmup 3 > $D/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vlut_mpgemm32_kernel -s 6 -c 1 -o $D/k132_full python bench.py --profile --steps 4 --warmup 3 > $D/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vlut_mpgemm32_sk -s 2 -c 1 -o $D/sk32_full python scripts/prof_one.py 3072 23040 256 5 12 1 32 1 768 > $D/ncu_sk32.log 2>&1
timeout 1500 python bench.py --table $D/configs.csv > $D/table.log 2>&1
