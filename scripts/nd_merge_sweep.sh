# coarse ND solve time per merge schedule (nd_levels.py prints the whole-solve line first)
cfgs=${1:-"4 3"}
for cfg in $cfgs; do
  for s in "" "2,2,3,3,5" "2,2,3,4,4" "2,2,4,4,3" "2,3,3,3,4" "2,2,3,3,3,2" "3,3,3,3,3" "2,2,2,3,3,3" "2,3,3,4,3"; do
    python scripts/nd_levels.py $cfg $s 2>&1 | grep "whole solve" | sed "s/^/cfg $cfg /"
  done
done
