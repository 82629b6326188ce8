for n in 300 400 512 700; do
  for g in 0 38 75 100 128; do
    if [ $g = 0 ]; then unset STO_REG_GRID; else export STO_REG_GRID=$g; fi
    echo "grid=$g $(timeout 60 python tools/midsize_sweep.py $n 2>&1 | tail -1)"
  done
done
