# A/B of library builds on one box (FASTH_LIB), alternating processes:
#   bash scripts/lib_ab.sh rounds lib/a.so lib/b.so [lib/c.so ...]
N=$1; shift
for i in $(seq $N); do
  for L in "$@"; do echo "== $L"; FASTH_LIB=$L timeout 200 python scripts/step_env.py base 2>/dev/null | grep variant; done
done
