# loss-head accumulators in registers: loss/step tests, repeatability, kernel A/B vs exp/ls0.so
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_train_gpu.py tests/test_probes_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/race_step.py 20 2 2>&1 | tail -1
KGREP="GPU kernel|loss_" bash scripts/gpu_var.sh ls0
