TAG=r03r bash scripts/gpu_evidence_r03.sh 2>&1 | tail -45
TAG=r03r REPS=10 bash scripts/checked_run.sh 2>&1 | tail -20
