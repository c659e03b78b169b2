cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QPINN_VERBOSE=1 timeout 900 python -m pytest tests/test_train_gpu.py -q -p no:cacheprovider -s > gpurun_out/train_tests.log 2>&1; tail -15 gpurun_out/train_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
python scripts/profile_step.py > gpurun_out/prof_step.txt 2>&1; head -30 gpurun_out/prof_step.txt
