RAS3_VARIANTS=col:2,cl2p:3,cl2t:3 timeout 300 python tools/ras3_probe.py 128 5
RAS3_VARIANTS=cl2p:3,cl2t:3 timeout 300 python tools/ras3_probe.py 512 3
