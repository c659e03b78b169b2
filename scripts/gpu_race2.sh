cd $GRAFT_REPO_ROOT
echo "== serial side stream"; QPINN_SERIAL_BWD=1 timeout 600 python scripts/race_check.py 60 2>&1 | grep -E "repeats differ"
echo "== launch blocking"; CUDA_LAUNCH_BLOCKING=1 timeout 600 python scripts/race_check.py 60 2>&1 | grep -E "repeats differ"
echo "== racecheck"; timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/race_small.py 4096 2>&1 | tail -25
echo "== synccheck"; timeout 600 compute-sanitizer --tool synccheck python scripts/race_small.py 4096 2>&1 | tail -15
echo "== memcheck"; timeout 600 compute-sanitizer --tool memcheck python scripts/race_small.py 4096 notan 2>&1 | tail -15
