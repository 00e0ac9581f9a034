for s in "64 129 7 0 0" "115 129 16 0 0" "115 129 16 1 1" "115 200 16 1 1" "115 129 12 1 1" "15 129 7 4 8" "115 160 7 0 0" "32 129 7 0 0"; do
  echo -n "$s : "; python tools/check_shape.py $s 2>&1 | grep loglik
done
