mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r2l.txt 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_r2l.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2l.txt 2>&1
python bench.py --extras c2 > gpurun_out/bench_r2l.jsonl 2> gpurun_out/bench_r2l.err
