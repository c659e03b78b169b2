cd $GRAFT_REPO_ROOT
timeout 900 python scripts/race_gemm.py 150 2>&1 | tail -30
