# One gpurun round trip for a tag: GPU tests, smoke, default bench, reference arm, ncu launch list + full capture.
# Usage (from the repo root): gpurun --timeout 2700 -- 'bash profiles/gcall.sh r2k'
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.txt 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
python bench.py > gpurun_out/bench_$TAG.jsonl 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.jsonl 2> gpurun_out/bench_ref_$TAG.err
bash profiles/prof.sh $TAG > gpurun_out/prof_$TAG.out 2>&1
