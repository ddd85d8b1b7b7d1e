for kv in "4 16" "2 16" "1 16" "4 8" "4 32" "2 8" "8 16"; do set -- $kv
  echo "near $1 chunk $2"; ZOLO_DAG_NEAR=$1 ZOLO_DAG_CHUNK=$2 python tools/quick_check.py cfg3 2>&1 | grep -E "apply_filter" | tail -1 | cut -c1-120
done
