cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 0 1; do
  if [ $v = 1 ]; then export SB_GRAPH=1; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('graph=$v ms %.3f e2e %.0f' % (d['ms_per_step'], d['e2e']['value']))"
done
