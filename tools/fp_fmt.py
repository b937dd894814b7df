import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    if "stages" in d:
        g=d["stages"]; h=d["host"]
        print(d["step"], d["s"], {k:(g[k],h.get(k)) for k in g if g[k]>60 and k not in ("optdmd.basis","optdmd.modes_total")})
    else: print(d)
