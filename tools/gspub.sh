#!/bin/bash
# wavefront GS: rows per cross-CTA flag release (kGsPub) 4 (default) vs 1, 2
for L in paper_1208_1975_b200/libpsmooth.so tools/libpsmooth_pub1.so tools/libpsmooth_pub2.so; do
  echo "lib=$L" >> gpurun_out/gspub.log
  PSM_LIB=$PWD/$L timeout -s KILL 300 python tools/bench_configs.py --only C2,C4 --runs 1,0 2>&1 | cut -c150-260 >> gpurun_out/gspub.log
done
