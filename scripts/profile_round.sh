# Full evidence set for a round: bench line, ncu launch list of a short bench run, and one
# ncu --set full capture of a sparse block step.  Usage: bash scripts/profile_round.sh <tag>
TAG=${1:-r01}
set -x
python bench.py > gpurun_out/bench_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --kernel-reps 2 \
    --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/sparse_$TAG python scripts/profile_step.py --only sparse > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/dense_$TAG python scripts/profile_step.py --only dense > /dev/null 2>&1
ls -la gpurun_out | tail -8
