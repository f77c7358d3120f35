cd $GRAFT_REPO_ROOT
for shape in "--cin 16 --cout 16" "--cin 48 --cout 16" "--cin 32 --cout 32 --h 544 --w 960"; do echo "== $shape"; NAR_B200_LIB=scripts/exp/trace.so timeout 120 python scripts/tc_trace.py $shape 2>&1 | tail -17; echo "== $shape debug 8+1+4 (MMA only)"; NAR_B200_LIB=scripts/exp/trace.so timeout 120 python scripts/tc_trace.py $shape --debug 13 2>&1 | tail -8; done
