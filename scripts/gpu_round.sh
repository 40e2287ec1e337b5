timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2_gputest5.log
for s in "6912 2560 128 4" "6912 2560 64 4" "3072 23040 128 4" "3072 23040 64 5" "3072 23040 128 5"; do
  timeout 300 python scripts/kbench.py --shape $s >> gpurun_out/r2_nvalley.txt 2>&1
done
