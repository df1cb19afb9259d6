"""Median per-phase cycle counts of a tools/tc_trace.py timeline (steady state)."""
import sys
import numpy as np

N = "u P X1 X2 G1s G1w G1c G2s G2w G2c STf STr Es Et Ed Ea Ec Eb Ee h0l h0e h1l h1e cs".split()
for f in sys.argv[1:]:
    L = [l.split() for l in open(f) if l.strip() and l.split()[0].isdigit()]
    a = np.array([[int(x) for x in l] for l in L])[10:]
    c = {k: i for i, k in enumerate(N)}
    m = lambda x, y: int(np.median(a[:, c[y]] - a[:, c[x]]))
    print(f, "tiles", len(a), "cycles/tile", int(np.median(np.diff(a[:, c['P']]))),
          "| epi: Es->Et", m('Es', 'Et'), "Et->Ed", m('Et', 'Ed'), "Ed->Ea", m('Ed', 'Ea'), "Ea->Ec", m('Ea', 'Ec'),
          "Ec->Eb", m('Ec', 'Eb'), "Eb->Ee", m('Eb', 'Ee'), "idle", int(np.median(a[2:, c['Es']] - a[:-2, c['Ee']])),
          "| P->Et", m('P', 'Et'), "P->STr", m('P', 'STr'), "G1s->G1w", m('G1s', 'G1w'), "G1w->c", m('G1w', 'G1c'),
          "G2s->G2w", m('G2s', 'G2w'), "G2w->c", m('G2w', 'G2c'), "Ec->STf", m('Ec', 'STf'), "STf->STr", m('STf', 'STr'))
    if a.shape[1] > 19:
        print("   Ea->h0l", m('Ea', 'h0l'), "h0l->h0e", m('h0l', 'h0e'), "h0e->h1l", m('h0e', 'h1l'), "h1l->h1e", m('h1l', 'h1e'),
              "h1e->cs", m('h1e', 'cs'), "cs->Ec", m('cs', 'Ec'))
