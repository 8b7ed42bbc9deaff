python tools/gpu/claim_ab.py
for cl in 2000 6000 20000; do WPM_CLAIM_LOW=$cl python -c "
import sys, os; sys.path.insert(0, os.getcwd()); sys.argv=['x']
exec(open('tools/gpu/claim_ab.py').read().split('for n in')[0])
import json
for n in (5, 8, 11): print(json.dumps(run(n, 'claim')))
"; done
