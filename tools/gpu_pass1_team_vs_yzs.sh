#!/bin/bash
# pass 1: team mapping vs the YZS path (MNL_NO_YZW) on a few shapes
for shp in "200000 50 30 10 5" "400000 10 20 4 2" "400000 16 20 4 2" "400000 30 10 4 2" "1000000 4 3 2 1" "200000 64 30 10 5"; do
  python tools/time_pass1.py $shp | tail -1
  MNL_NO_YZW=1 python tools/time_pass1.py $shp | tail -1
done
