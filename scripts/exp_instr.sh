cd $GRAFT_REPO_ROOT
echo "== normal"; python scripts/probe/run_instr.py
echo "== debug 66 (no fusion compute)"; KMD_DEBUG=66 python scripts/probe/run_instr.py
echo "== debug 34 (no field compute)"; KMD_DEBUG=34 python scripts/probe/run_instr.py
