import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print({k: round(v["ms_new"],3) for k,v in d.items() if k.startswith("step")})
