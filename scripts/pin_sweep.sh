for mb in 0 1 10 20 30; do
  echo "== B200IPC_L2_PIN_MB=$mb"
  B200IPC_L2_PIN_MB=$mb python scripts/mas_probe.py 2>&1 | grep -E "block-jacobi|mas pcg levels=1"
done
