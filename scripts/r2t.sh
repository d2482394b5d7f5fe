set -u
python -m pytest tests/test_gpu_contacts.py tests/test_gpu_ccd.py tests/test_gpu_fullsize.py tests/test_gpu_stepper.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -2
for v in old g8 g16 g32; do
  if [ $v = g16 ]; then unset B200IPC_LIB; else export B200IPC_LIB=$PWD/scripts/probes/_bin/libb200ipc_$v.so; fi
  echo "== $v"
  python bench.py --skip-cpu 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); n=d['newton']
print('broad', round(n['broad_phase_ms'],3), 'narrow', round(n['narrow_phase_ms'],3), 'ccd', round(n['ccd']['sweep_plus_filter_ms'],3), 'e2e', round(n['newton_direction_e2e']['ms'],2), round(n['newton_direction_e2e_mas']['ms'],2), 'steps', [round(s['wall_ms'],1) for s in n['time_step']['steps']])
c=d.get('newton_config2') or d.get('newton_sphere') or {}
print({k: round(v,3) for k,v in c.items() if k in ('broad_phase_ms','narrow_phase_ms','detect_ms')})
"
done
