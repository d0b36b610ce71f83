cd $GRAFT_REPO_ROOT
timeout 600 python tools/overlap_probe.py 2>&1 | tail -1
PRIO=-1,0 timeout 600 python tools/overlap_probe.py 2>&1 | tail -1
PRIO=0,-1 timeout 600 python tools/overlap_probe.py 2>&1 | tail -1
