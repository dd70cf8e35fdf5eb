cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SB_PLACE_TIMES=1 python bench.py --config c2_mixed --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/pt.json 2> gpurun_out/pt.err
tail -26 gpurun_out/pt.err
SB_ROUND_DEBUG=1 python bench.py --config c2_mixed --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/pt2.json 2> gpurun_out/pt2.err
tail -2 gpurun_out/pt2.err
