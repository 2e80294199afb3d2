# multigrid variants on the configs[1] sweep positions (k = 8)
export PRECONDS=amg
for cfg in "1 1.5 1" "0 1.5 1" "1 1.0 0" "1 1.5 0"; do set -- $cfg
  echo "== f32=$1 oc=$2 w=$3"
  ECT_AMG_F32=$1 ECT_AMG_OC=$2 ECT_AMG_WCYCLE=$3 timeout 300 python scripts/amg_gpu_probe.py 8 1e-8 2>&1 | grep -v "^Exception\|Traceback\|File\|Attribute"
done
for k in 2 16; do
  echo "== default k=$k"
  timeout 300 python scripts/amg_gpu_probe.py $k 1e-8 2>&1 | grep -v "^Exception\|Traceback\|File\|Attribute"
done
