# end-of-round-2 refresh after the g = 4 K1-32-SK table-buffer change
set -x
D=gpurun_out/r02f4
mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q > $D/gputests.txt 2>&1
timeout 600 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 1500 python bench.py --table $D/configs.csv > $D/table.log 2>&1
