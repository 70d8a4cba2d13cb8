# Timing of library variants (build them with -DSPGEMM_REUSE_U=.. -DSPGEMM_REUSE_MINB=.. into
# lib/libspgemm_b200_<name>.so first); run under gpurun.
cd $GRAFT_REPO_ROOT/paper_2206_07244_b200/lib
cp libspgemm_b200.so base.so
for v in base u2_b5 u8_b4 u4_b4; do
  if [ $v = base ]; then cp base.so libspgemm_b200.so; else cp libspgemm_b200_$v.so libspgemm_b200.so; fi
  cd $GRAFT_REPO_ROOT; echo "== $v"; timeout 200 python tools/quick_timing.py 2 2>&1 | tail -1; cd paper_2206_07244_b200/lib
done
cp base.so libspgemm_b200.so
