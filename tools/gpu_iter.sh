cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
for e in 17 21 25 31; do echo "E=$e"; MCR_XDOT_E=$e timeout 300 python tools/prof_xdot.py c2 2; done > $O/e_sweep2.log 2>&1
