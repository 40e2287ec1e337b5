mkdir -p gpurun_out/r02g
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02g/gputests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02g/smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g/bench.json 2> gpurun_out/r02g/bench.err
