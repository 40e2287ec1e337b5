mkdir -p gpurun_out/mc
timeout 600 python -m pytest tests -m gpu -q -k "multicast or allgather or peer_outputs" -rs > gpurun_out/mc/tests.txt 2>&1
