# Profiling recipe for the round's evidence (run on the GPU box from the repo
# root, one ncu per gpurun call):  bash profiles/capture.sh list | full
set -e
CMD="python bench.py --n 512 --axes z --steps 1 --warmup 0 --no-e2e --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_z.log 2>&1   # the same command exits 0 without ncu first
case "$1" in
  list) ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
          --log-file gpurun_out/launches512.csv $CMD > gpurun_out/ncu_list.log 2>&1 ;;
  full) timeout 1200 ncu --set full --import-source on --clock-control none \
          -k regex:"k_stencil_ph|k_fwd_c2|k_thomas_x|k_inv_c2" -s 7 -c 4 \
          -o gpurun_out/prof512 -f $CMD > gpurun_out/ncu_full.log 2>&1 ;;
esac
