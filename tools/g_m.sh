mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/m_default.txt 2>&1
timeout 600 python bench.py --workload c3 --steps 2 --warmup 2 --no-cpu > gpurun_out/m_c3.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_ref.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1
