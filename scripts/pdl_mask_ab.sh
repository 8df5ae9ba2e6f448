for v in 0 31 7 3 24 23; do echo -n "mask=$v "; BDDC_PDL_PCG=$v python bench.py --no-mode-b --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['pcg_only_it_per_s'],1))"; done
