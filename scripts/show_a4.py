import sys, json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
shapes=sorted({(r['M'],r['N'],r['KP']) for r in rows}, key=lambda x:(x[2],-x[0]*x[1]))
tags=[]
[tags.append(r['tag']) for r in rows if r['tag'] not in tags]
print('shape'.ljust(22), *[t.ljust(16) for t in tags])
for s in shapes:
    cells=[]
    for t in tags:
        r=[r for r in rows if r['tag']==t and (r['M'],r['N'],r['KP'])==s]
        cells.append((f"{r[0]['us']:7.1f}us {r[0]['frac']:.3f}" if r else "-").ljust(16))
    print(str(s).ljust(22), *cells)
