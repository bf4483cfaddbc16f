for d in 1 2 3 5 8 16; do
  echo "depth $d"
  SPQR_SPEC_DEPTH=$d SPQR_PROF=1 REPS=3 timeout 300 python tools/time_c2.py 2>&1 | grep -E "^\[spqr prof\] sparsify_cols |scols.upload|'t_factorize'|nW" | grep -oE "sparsify_cols +[0-9.]+ s|upload\+cpqr\+fetch +[0-9.]+ s|'t_factorize': np.float64\([0-9.]+\)|nW [0-9]+ nnz_w [0-9]+" | tr '\n' ' '
  echo
done
