# developer: n = 15 look-ahead / policy / configuration around the default (configuration 1)
for r in 1 2 3; do
  for L in 3 4 5 6 8; do echo -n "L=$L "; PTDR_L=$L timeout 120 python tools/diag_n15.py 15 2>&1 | tail -1; done
  for P in fnl flf fnu; do echo -n "pol=$P "; PTDR_POL=$P timeout 120 python tools/diag_n15.py 15 2>&1 | tail -1; done
  echo -n "cfg=8 "; PTDR_PIPE_CFG=8 timeout 120 python tools/diag_n15.py 15 2>&1 | tail -1
done
