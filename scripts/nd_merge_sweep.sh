# coarse ND solve time per merge schedule (nd_levels.py prints the whole-solve line first)
for cfg in 4 3; do
  for s in "" "2,3,3,3,3,3" "1,3,3,3,3,4" "2,2,3,3,3,4" "3,3,3,4,4" "4,4,4,5" "2,3,3,4,5" "2,4,4,4"; do
    python scripts/nd_levels.py $cfg $s 2>&1 | grep "whole solve" | sed "s/^/cfg $cfg /"
  done
done
