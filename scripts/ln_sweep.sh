# LayerNorm backward launch-shape sweep (bf16-dy form, C2 rows): nst warps smem-cap-KB blocks-per-SM
for cfg in "2 4 110 2" "3 4 150 1" "2 2 110 4" "1 4 110 4" "2 4 160 1" "3 2 110 3" "1 2 60 8" "2 1 60 8" \
           "3 4 130 1" "2 4 90 2" "3 2 80 3" "4 2 110 2" "2 3 90 2" "1 4 60 5"; do
  set -- $cfg
  echo "nst=$1 warps=$2 cap=$3 persm=$4: $(P2R_LN_BWD_NST=$1 P2R_LN_BWD_WARPS=$2 P2R_LN_BWD_SMEM_KB=$3 P2R_LN_BWD_PERSM=$4 python scripts/ln_bench.py | head -1)"
done
