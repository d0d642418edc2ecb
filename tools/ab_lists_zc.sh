# A/B of the sampled launch's index lists: zero-copy from pinned staging (default) vs copied first
for i in 1 2 3; do
  for zc in 0 1; do
    echo "== BT_LISTS_ZC=$zc"
    BT_LISTS_ZC=$zc python bench.py --steps 20 --warmup 5 --no-bert 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('device', d['value'], 'e2e', d['e2e']['value'], 'run_minibatch', d.get('run_minibatch'))"
  done
done
