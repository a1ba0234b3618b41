import json,sys
for f in sys.argv[1:]:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["ms_per_step"],4), round(d["value"],1), "collect", round(d["roofline"]["frac"],3), "select", round(d["select_stage"]["ms"],4), round(d["select_stage"]["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("parity"))
