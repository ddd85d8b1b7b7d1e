for kv in "4 16" "4 24" "4 12" "2 20" "6 20"; do set -- $kv
  echo "near $1 chunk $2"; ZOLO_DAG_NEAR=$1 ZOLO_DAG_CHUNK=$2 python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter" | sed -n '2p;4p' | cut -c1-120
done
