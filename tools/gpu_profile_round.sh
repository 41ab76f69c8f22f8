#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}  # device-sized levels
# Round evidence: bench (both arms), per-config timings, launch lists, full
# ncu captures of the top kernels, the 2-rank fused-halo path on one GPU.
# Outputs under gpurun_out/round/.
# PART (first argument): 1 = bench, configs, launch lists, smoke; 2 = ncu of
# the line-GS and band kernels; 4 = ncu of the plane-GS kernels; 3 = ncu of box, line Jacobi and
# zgen kernels plus the 2-rank fused-halo run (each part's outputs stay under
# gpurun's 64 MiB copy-back limit); default all.
PART=${1:-all}
O=gpurun_out/round; mkdir -p $O
make -j all > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
if [ "$PART" = all ] || [ "$PART" = 1 ]; then
timeout -s KILL 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference > $O/bench_ref.json 2>&1; echo "ref rc=$?"
timeout -s KILL 900 python tools/bench_configs.py > $O/configs.jsonl 2>&1; echo "configs rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1
for c in C1 C2 C3 C4 F1 F3; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python tools/bench_configs.py --only $c --steps 1 --warmup 1 > /dev/null 2>&1
  python tools/launch_summary.py $O/launches_$c.csv > $O/launches_$c.txt 2>&1
done
# C2: one multi-sweep launch (10 GS sweeps) of the pipelined line-GS kernel
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2_10.csv \
  python tools/bench_configs.py --only C2 --steps 10 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_C2_10.csv > $O/launches_C2_10.txt 2>&1
timeout -s KILL 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"
fi
if [ "$PART" = all ] || [ "$PART" = 2 ]; then
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:line_gs_pipe -s 1 -c 1 \
  -o $O/gs_multi_256 python tools/bench_configs.py --only C2 --runs 1 --steps 10 --warmup 1 > /dev/null 2>&1
echo "ncu gs rc=$?"
bash tools/ncu_plane.sh 512 round/plane_band_512 > /dev/null 2>&1; echo "ncu band rc=$?"
for r in gs_multi_256 plane_band_512; do python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
fi
if [ "$PART" = all ] || [ "$PART" = 4 ]; then
bash tools/ncu_plane_gs.sh round/pgs > $O/pgs.txt 2>&1; echo "ncu plane gs rc=$?"
fi
if [ "$PART" = all ] || [ "$PART" = 3 ]; then
bash tools/ncu_box.sh 512 8 round/box_8_512 > /dev/null 2>&1; echo "ncu box rc=$?"
bash tools/ncu_line.sh 1024 round/line_jacobi_1024 > /dev/null 2>&1; echo "ncu line rc=$?"
bash tools/ncu_line.sh 512 round/line_jacobi_512 > /dev/null 2>&1; echo "ncu line512 rc=$?"
bash tools/ncu_zgen.sh round/line_zgen_f3 > /dev/null 2>&1; echo "ncu zgen rc=$?"
# C1: the 64^3 line-Jacobi sweep (latency-bound small patch)
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:line_jacobi_nx -s 5 -c 1 \
  -o $O/line_c1_64 python tools/bench_configs.py --only C1 --runs 0 --steps 10 --warmup 1 > /dev/null 2>&1
echo "ncu c1 rc=$?"
# the fused peer-memory halo: 2 ranks sharing this one GPU (IPC), gloo for the plumbing
PSM_HALO=p2p PSM_DIST_BACKEND=gloo timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 --shape 512 512 512 \
  --no-cpu-baseline > $O/bench_p2p_2ranks_1gpu.json 2> $O/bench_p2p.err; echo "p2p rc=$?"
for r in box_8_512 line_jacobi_1024 line_jacobi_512 line_zgen_f3 line_c1_64; do
  python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1
done
fi
echo done
