export PRECONDS=amg
for cfg in "1.0 0" "1.0 1" "1.5 1"; do set -- $cfg
  echo "== configs[1] k=8 oc=$1 w=$2"
  ECT_AMG_OC=$1 ECT_AMG_WCYCLE=$2 timeout 300 python scripts/amg_gpu_probe.py 8 1e-8 2>&1 | grep -v "^Exception\|Traceback\|File\|Attribute"
done
