import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    ks = " ".join(f"{k}={v.get('ms_per_step', v.get('ms_per_launch', 0))*1e3:.1f}" for k, v in d.get("kernels", {}).items())
    print(f.split('/')[-1], round(d["value"]), d["unit"], f"{d['ms_per_step']*1e3:.1f}us/step", ks)
