export PATCHSMOOTH_MAX_CELLS=100000000000
mkdir -p gpurun_out
bash tools/ncu_plane_gs.sh prof_pgs3 2>&1 | grep -E "==|Duration|Eligible|Issue Slots"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:line_gs_pipe -s 1 -c 1 \
  -o gpurun_out/prof_gsm python tools/bench_configs.py --only C2 --runs 1 --steps 10 --warmup 1 > gpurun_out/prof_gsm.log 2>&1
echo "gsm rc=$?"
python tools/ncu_summary.py gpurun_out/prof_gsm.ncu-rep 2>&1 | head -50
