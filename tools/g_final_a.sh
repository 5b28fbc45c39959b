mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fa_smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fa_tests.txt 2>&1; echo rc=$? >> gpurun_out/fa_tests.txt
