mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2r_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2r_all.txt 2>&1; echo "rc=$?" >> gpurun_out/r2r_all.txt
timeout 900 python bench.py > gpurun_out/r2r_bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2r_ref.txt 2>&1
