# development: nested-dissection leaf size vs sweep / factorization speed on a config
# usage: bash tools/dev/leaf_sweep.sh cfg3 "64 96 128 192"
for leaf in ${2:-128 160 192 224 256 320}; do
  echo "== leaf $leaf"; ND_LEAF=$leaf python tools/quick_check.py ${1:-cfg3} 2>&1 | grep -E "factor wall|apply_filter" | tail -2 | cut -c1-175
done
