# Round-2 config-4/5 sweeps only (re-run after the last GEMM change) -> profiles/r02/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1200 python scripts/sweep_ablation.py 5 > $O/config4_ablation_dielectric.jsonl 2> $O/config4.err
timeout 2700 python scripts/sweep_pqc.py --all-ansatze > $O/config5_sweep.jsonl 2> $O/config5.err
wc -l $O/config5_sweep.jsonl $O/config4_ablation_dielectric.jsonl
