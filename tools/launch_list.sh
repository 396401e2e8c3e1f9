# launch list (ncu gpu__time_duration per kernel, cold-cache, serialised) of one solve:
#   bash tools/launch_list.sh OUT [CONFIG] [SKIP] [COUNT]   -> gpurun_out/OUT.csv
out=$1; cfg=${2:-c4}; skip=${3:-60}; cnt=${4:-120}
TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none -s "$skip" -c "$cnt" --csv \
  --log-file "gpurun_out/$out.csv" python tools/step.py --config "$cfg" --solves 1 > "gpurun_out/$out.log" 2>&1
echo "launch list $out rc=$?"
