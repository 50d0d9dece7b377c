# Per-config device time per time step on one GPU (profiles/r*_configs_1gpu.txt): bash tools/all_configs.sh
for c in "C0 strang 200" "C0 if4 200" "C1 strang 400" "C1 split4 400" "C1 if4 400" "C2 split4 20" "C2 if4 20" "C3 if4 10" "C3 strang 10" "C4 if4 8"; do
  set -- $c
  r=$(timeout 900 python tools/run_config.py $1 $2 $3 2>/dev/null | tail -1)
  echo "$1 $2 $3 $r"
done
