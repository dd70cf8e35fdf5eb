cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_mixed or relations_variants or hole or c1_tabletop" 2>&1 | tail -3
for c in 1 2 4 8; do
  SB_CLUSTER=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cluster $c ms %.3f' % d['ms_per_step'], 'per_inst %.3f fast %.3f' % (d['phase_profile_per_step']['ev_per_instance_ms'], d['phase_profile_per_step']['ev_fast_ms']))"
done
