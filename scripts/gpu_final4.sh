# end-of-round-2 final artifacts (after the >= 2 CTAs-per-tile meeting rule)
set -x
D=gpurun_out/r02f5
mkdir -p $D
timeout 600 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 1500 python bench.py --table $D/configs.csv > $D/table.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --profile --steps 4 --warmup 3 > $D/ncu_launch.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.txt 2>&1
