import sys, numpy as np, json
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2506_13624_b200 as B
z=np.load('tests/golden/cfg4_population.npz')
ctx=B.Context(0)
spec=B.intersection_spec(63,10.0,0.1)
off=z['rec_off']
def lev(a):
    a=np.asarray(a); o=np.full(a.shape,-1,np.int8); ok=a>0; o[ok]=np.rint(-np.log2(a[ok])); return o
for i in [496,568,1441,1602,1787,2278,3127, 601]:
    p=B.build_intersection_case(spec,2,2,perturb_seed=42+i)
    r=B.solve(p, max_records=1000, ctx=ctx)
    # FIFO single-instance batch, 64x8 and 256x1
    out=[]
    for shape in [(256,1),(64,8)]:
        bt=B.Batch(ctx,[p],max_records=1000); bt.set_models(); bt.set_launch(*shape); bt.solve(); reps,_=bt.results()
        out.append(reps[0].inner_iterations)
    g=lev(r.report.iterations['alpha']); ref=z['rec_level'][off[i]:off[i+1]]
    n=min(len(g),len(ref)); d=np.flatnonzero(g[:n]!=ref[:n])
    print(i,'single',r.report.inner_iterations,'batches',out,'ref',z['inner'][i],'first diff rec',d[:1], 'nrec',len(g),len(ref))
