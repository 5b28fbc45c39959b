# usage (on the GPU box): bash tools/gpu_check.sh TAG
# smoke, the whole -m gpu suite and the default bench line (all blocks), in that order
T=${1:-chk}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.txt
