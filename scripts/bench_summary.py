import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): continue
    d=json.loads(line)
    c=d["config"]
    print(c["code"], c["k"], "B=%d"%c["batch"], "impl", c["matvec_impl"], "value", d["value"], "ms", d["ms_per_step"], "gemv", d["roofline"]["achieved"], {k: v["us_per_layer"] for k, v in c["per_layer"].items()})
