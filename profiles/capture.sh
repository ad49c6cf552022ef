# Profiling recipe for the round's evidence (run on the GPU box from the repo
# root):  bash profiles/capture.sh list | full | both | f32
set -e
CMD="python bench.py --n 512 --axes z --steps 1 --warmup 0 --no-e2e --no-cpu"
CMD32="python bench.py --n 512 --axes z --steps 1 --warmup 0 --no-e2e --no-cpu --precision f32"
mkdir -p gpurun_out
if [ "$1" = f32 ]; then
  $CMD32 > gpurun_out/plain_z32.log 2>&1   # the same command exits 0 without ncu first
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches512_f32.csv $CMD32 > gpurun_out/ncu_list32.log 2>&1
  timeout 1200 ncu --set full --import-source on --clock-control none \
      -k regex:"k_stencil_pht|k_fwd_q|k_zsolve_tma|k_inv_q" -s 8 -c 4 \
      -o gpurun_out/prof512_f32 -f $CMD32 > gpurun_out/ncu_full32.log 2>&1
  exit 0
fi
$CMD > gpurun_out/plain_z.log 2>&1   # the same command exits 0 without ncu first
if [ "$1" = list ] || [ "$1" = both ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches512.csv $CMD > gpurun_out/ncu_list.log 2>&1
fi
if [ "$1" = full ] || [ "$1" = both ]; then
  timeout 1200 ncu --set full --import-source on --clock-control none \
      -k regex:"k_stencil_pht|k_fwd_q|k_zsolve_tma|k_inv_q" -s 8 -c 4 \
      -o gpurun_out/prof512 -f $CMD > gpurun_out/ncu_full.log 2>&1
fi
