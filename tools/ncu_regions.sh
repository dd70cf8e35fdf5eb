cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_relation_regions -s 8 -c 2 -o gpurun_out/prof_regions -f python bench.py --steps 1 --warmup 1 --config c2_mixed --no-cpu-baseline > gpurun_out/prof_regions.log 2>&1
echo rc=$?
