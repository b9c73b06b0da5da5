cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in A B; do cp abso/$v.so paper_2508_05020_b200/libamr.so; echo -n "$v "; python scripts/time_stage.py weno5 2>&1 | tail -1; done; done
cp abso/B.so paper_2508_05020_b200/libamr.so
