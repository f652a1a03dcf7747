# End-of-round evidence: full GPU suite, smoke, two bench lines, ncu launch list + full
# captures of both steps (profile_round.sh), CUPTI step timelines.  usage: bash scripts/gpu_final.sh <tag>
TAG=${1:-r02h}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 bash scripts/profile_round.sh $TAG
timeout 300 python bench.py > gpurun_out/bench2_$TAG.log 2>&1
timeout 120 python scripts/step_timeline.py --kind sparse > gpurun_out/timeline_sparse_$TAG.txt 2>&1
timeout 120 python scripts/step_timeline.py --kind dense > gpurun_out/timeline_dense_$TAG.txt 2>&1
tail -1 gpurun_out/bench_$TAG.log | cut -c1-600
