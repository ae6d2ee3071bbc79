import sys, statistics as st
for fn in sys.argv[1:]:
    rows = []
    for l in open(fn):
        p = l.split()
        if len(p) > 12 and p[0].isdigit():
            nums = [int(x) for x in p if x.lstrip('-').isdigit()]
            # k phase we dep iss w h d issue ready done
            rows.append(nums)
    for ph in (0, 1):
        r = [x for x in rows if x[1] == ph and x[0] > 20]
        if not r: continue
        print(fn, 'phase', ph, 'n', len(r), 'wait_empty', st.median([x[2] for x in r]), 'dep', st.median([x[3] for x in r]),
              'issue', st.median([x[4] for x in r]), 'cons_wait', st.median([x[5] for x in r]), 'hold', st.median([x[6] for x in r]),
              'post', st.median([x[7] for x in r]))
    iss = [x[8] for x in rows]
    print('  cycles per tile (issue interval)', (iss[-1] - iss[20]) / (len(iss) - 21))
