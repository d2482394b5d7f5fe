set -u
for v in base pf; do
  lib=$PWD/scripts/probes/_bin/libb200ipc_$v.so
  echo "== $v"
  B200IPC_LIB=$lib python scripts/layout_probe.py stack 2>&1 | tail -3
  B200IPC_LIB=$lib python scripts/layout_probe.py sphere 2>&1 | tail -3
done
