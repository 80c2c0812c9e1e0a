# A/B of two library builds on one box (FASTH_LIB), alternating processes:
#   bash scripts/lib_ab.sh lib/a.so lib/b.so [rounds]
A=$1; B=$2; N=${3:-3}
for i in $(seq $N); do
  for L in $A $B; do echo "== $L"; FASTH_LIB=$L timeout 200 python scripts/step_env.py base 2>/dev/null | grep variant; done
done
