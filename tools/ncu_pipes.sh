#!/bin/bash
# Tensor (DMMA) / fp64 pipe utilisation and DRAM bytes of every kernel in one
# step of a config: tools/ncu_pipes.sh CONFIG RUNIDX OUT
CFG=${1:-C3}; RUN=${2:-1}; OUT=${3:-pipes}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/$OUT.csv \
  python tools/bench_configs.py --only $CFG --runs $RUN --steps 1 --warmup 1 > /dev/null 2>&1
python - gpurun_out/$OUT.csv <<'PY'
import csv, sys, collections
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows)); h = r[0]
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for x in r[1:]:
    d = dict(zip(h, x))
    k = d["Kernel Name"][:60]
    try:
        agg[k][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    except ValueError:
        pass
for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
    t = m.get("gpu__time_duration.sum", [0])
    if "psm" not in k and "gemm" not in k:
        continue
    n = len(t)
    avg = lambda name: sum(m.get(name, [0])) / max(1, len(m.get(name, [0])))
    print(f"{k:60s} n={n:4d} t_avg={sum(t)/n/1e3:9.1f}us dmma%={avg('smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"fp64%={avg('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"dram_GB={(avg('dram__bytes_read.sum') + avg('dram__bytes_write.sum'))/1e9:7.3f}")
PY
