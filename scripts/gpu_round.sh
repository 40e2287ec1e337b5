timeout 600 python scripts/chain_check.py 4 > gpurun_out/r2_chain.txt 2>&1
VLUT_NO_K32=1 timeout 600 python scripts/chain_check.py 4 >> gpurun_out/r2_chain.txt 2>&1
