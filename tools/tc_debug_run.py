import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_1808_04473_b200 as dbp
from paper_1808_04473_b200.synth import synth_frames
H,Y,S,n0 = synth_frames(1, 2, 1200, 14, 128, 16, 'qam16', [10.0, 10.0])
const = dbp.make_constellation('qam16')
Hd=torch.from_numpy(H).cuda(); Yd=torch.from_numpy(Y).cuda()
det = dbp.Detector('pd','lmmse',Hd.shape[0],128,16,14,[32]*4,const)
for i in range(3): det.run(Hd,Yd,float(n0[0]))
torch.cuda.synchronize()
