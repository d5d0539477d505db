cd /root/repo
export TFS_ALLOW_VARIANT_LIB=1
for rep in 1 2; do for w in X Z; do
 for cfg in "base TFS_PDL=0" "base TFS_PDL=1" "variants/pdl_notrig.so TFS_PDL=1"; do
  set -- $cfg; if [ $1 = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$1; fi
  steps=100; [ $w = Z ] && steps=20
  env $2 timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
  python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
print('$cfg $w', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']/1e6,2))"
 done; done; done
