cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/quick_timing.py 3 2 2>&1 | grep cfg
