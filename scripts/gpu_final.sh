# round-2 measurement artifacts (bench line, ncu launch list, full K1-32 capture,
# §8(d) table, K2 decode capture and decode sweep, GPU tests)
set -x
mkdir -p gpurun_out/r02f
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02f/gputests.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f/launches.csv python bench.py --profile --steps 4 --warmup 3 > gpurun_out/r02f/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vlut_mpgemm -s 6 -c 1 -o gpurun_out/r02f/k1_full python bench.py --profile --steps 4 --warmup 3 > gpurun_out/r02f/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vlut_slot -s 2 -c 1 -o gpurun_out/r02f/k2_decode python scripts/prof_decode.py > gpurun_out/r02f/ncu_k2.log 2>&1
timeout 600 python scripts/decode_bench.py > gpurun_out/r02f/decode.txt 2>&1
timeout 1500 python bench.py --table gpurun_out/r02f/configs.csv > gpurun_out/r02f/table.log 2>&1
