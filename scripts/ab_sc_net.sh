for sc in 18:3 18:6 18:9 18:18 16:8 24:6; do
  S=${sc%%:*}; C=${sc##*:}
  echo -n "S=$S C=$C "
  SMC_SW_S=$S SMC_SW_C=$C timeout 300 python scripts/variant_boundary.py 64,512,40000 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('v4 %.3g' % d['v4'], d['v4_cfg'])"
done
