mkdir -p gpurun_out/p16
for c in "3072 23040 16 4 2" "3072 23040 16 5 2" "3072 23040 64 4 2"; do
  echo "== $c"; timeout 300 python scripts/slot_phase_timing.py $c 2>&1 | grep -v warning | grep -E "^(CTAs|entry|idx|table|loop|tile|arrived|stored)"
done > gpurun_out/p16/phase.txt 2>&1
