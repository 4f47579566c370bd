#!/bin/bash
# Round-2 ncu evidence (run on the GPU box from the repo root; outputs under
# gpurun_out/, summaries copied to profiles/ afterwards).
set -x
mkdir -p gpurun_out
for c in c1 c2 c3; do
  python tools/prof_session.py $c 20 > gpurun_out/prof_$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 400 --csv \
      --log-file gpurun_out/r02_launches_$c.csv python tools/prof_session.py $c 20 > /dev/null 2>&1
done
python tools/prof_session.py c4 2 > gpurun_out/prof_c4.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches_c4.csv python tools/prof_session.py c4 2 > /dev/null 2>&1
# Full sections: one iteration's kernels at c1 and c2 (after 4 warm-up
# iterations), the fp64 projection passes at c4.
ncu --set full --clock-control none --import-source on -s 64 -c 16 \
    -o gpurun_out/r02_c1_full python tools/prof_session.py c1 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -s 8 -c 2 \
    -o gpurun_out/r02_c2_gemm_full python tools/prof_session.py c2 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"row_update|col_partial|col_write" -s 3 -c 3 \
    -o gpurun_out/r02_c4_projections_full python tools/prof_session.py c4 2 > /dev/null 2>&1
ls -la gpurun_out
