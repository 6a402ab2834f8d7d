import os, sys, subprocess, json
cfgs=[]
for name in ["tiny7","tiny33"]:
    for layout in ["gather","inline"]:
        for tr in ["aqr","fp32"]:
            for vb in [-1,12,-2]:
                if layout=="inline" and tr=="aqr" and vb not in (-1,0): continue
                cfgs.append((name,layout,tr,vb))

for cfg in cfgs:
    r=subprocess.run([sys.executable,'tools/gpu/diag_one.py',*map(str,cfg)],capture_output=True,text=True,env=dict(os.environ,CUDA_LAUNCH_BLOCKING="1"))
    print(cfg, "OK" if "OK" in r.stdout else ("FAIL "+r.stderr.strip().splitlines()[-1][:150] if r.stderr.strip() else "FAIL"), flush=True)
