cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/quick_timing.py 1 2 4 2>&1 | grep cfg
SPGEMM_NO_WH=1 python tools/quick_timing.py 2 2>&1 | grep cfg
