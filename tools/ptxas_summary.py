import re,sys,subprocess
txt=open(sys.argv[1]).read()
cur=None
rows=[]
for line in txt.splitlines():
    m=re.search(r"Compiling entry function '(\S+)'",line)
    if m: cur=m.group(1); spill=''; continue
    m=re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads",line)
    if m and cur: spill=f"spill {m.group(1)}/{m.group(2)}"
    m=re.search(r"Used (\d+) registers",line)
    if m and cur:
        rows.append((cur,int(m.group(1)),spill)); cur=None
names=[r[0] for r in rows]
dem=subprocess.run(['c++filt'],input='\n'.join(names),capture_output=True,text=True).stdout.splitlines()
for (n,r,s),d in zip(rows,dem):
    d=re.sub(r'\(anonymous namespace\)::','',d)
    print(f"{r:4d} {s:14s} {d[:150]}")
