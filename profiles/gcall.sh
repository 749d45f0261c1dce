mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r2k.txt 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_r2k.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2k.txt 2>&1
python bench.py > gpurun_out/bench_r2k.jsonl 2> gpurun_out/bench_r2k.err
bash profiles/prof.sh r2k > gpurun_out/prof_r2k.out 2>&1
