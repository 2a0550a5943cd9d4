cd $GRAFT_REPO_ROOT
python scripts/probe/run_instr.py
