# ncu --set full (with source) of selected kernels of one c4 solve, under gpurun:
#   bash tools/ncu_kernel.sh NAME_REGEX SKIP COUNT OUT [CONFIG]
# e.g. bash tools/ncu_kernel.sh StResidRestrict 4 1 rr  -> gpurun_out/rr.ncu-rep
# (TMG_NO_COND_NODES=1: ncu cannot profile kernels inside conditional graphs)
re=$1; skip=$2; cnt=$3; out=$4; cfg=${5:-c4}
TMG_NO_COND_NODES=1 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$re" -s "$skip" -c "$cnt" \
  -f -o "gpurun_out/$out" python tools/step.py --config "$cfg" --solves 1 > "gpurun_out/$out.log" 2>&1
echo "ncu $out rc=$?"
