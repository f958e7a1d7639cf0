#!/bin/bash
cd $GRAFT_REPO_ROOT
VOXANIM_BAND_TRACE=1 VOXANIM_READBACK_BANDS=$BANDS timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_1911_06001_b200 as vx
lib, ctx = vx.vxa(), vx.context()
sc = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
buf = np.empty((sc.height, sc.width, 3), np.uint8)
lib.vxa_host_register(ctx, buf.ctypes.data, buf.nbytes)
for k in range(8):
    sc.evaluate(k/30.0); sc.render(precision=vx.VXA_FP32, rgb=buf)
" 2>&1 | tail -5
