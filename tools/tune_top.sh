for cfg in "16 24 96" "8 24 96" "16 48 96" "16 24 64" "16 12 96" "16 48 64"; do
  set -- $cfg
  r3=$(GN_TOP_CLUSTER=$1 GN_TOP_FRONTS=$2 GN_TOP_MIN_ROWS=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']*1e3,2), round(d['per_iter_ms']['refactor'],3))")
  r4=$(GN_TOP_CLUSTER=$1 GN_TOP_FRONTS=$2 GN_TOP_MIN_ROWS=$3 timeout 600 python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']*1e3,1), round(d['per_iter_ms']['refactor'],3))")
  echo "C=$1 fronts=$2 minrows=$3 | C3 $r3 | C4 $r4"
done
