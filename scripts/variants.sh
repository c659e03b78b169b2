# Kernel-variant loop: per-kernel step times for the in-tree library and each exp/<tag>.so
# (built by scripts/build_variant.py).  Usage: variants.sh "<kernel regex>" tag1 tag2 ...
cd $GRAFT_REPO_ROOT
pat=$1; shift
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/profile_step.py 2>&1 | grep -E "$pat|GPU kernel"
done
