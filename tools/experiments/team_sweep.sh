# Sweep of the team/bulk combine layout (LAMFAST_TEAM=<warps>,<entries per thread>;
# 0 = direct stores).  Usage: bash tools/team_sweep.sh [steps]
steps=${1:-20}
for v in 0 4,2 8,2 3,1 5,1 1,3 6,2 8,1 2,3; do
  echo -n "C4 team=$v "; LAMFAST_TEAM=$v python tools/run_steps.py --config C4 --steps $steps 2>&1 | tail -1
done
for v in 0 5,1 3,2 7,2 4,3 8,1; do
  echo -n "C3 team=$v "; LAMFAST_TEAM=$v python tools/run_steps.py --config C3 --steps $steps 2>&1 | tail -1
done
for v in 0 3,1 4,2 5,1; do
  echo -n "C2 team=$v "; LAMFAST_TEAM=$v python tools/run_steps.py --config C2 --steps 50 2>&1 | tail -1
done
