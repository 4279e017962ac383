import sys
sys.path.insert(0, '.')
sys.argv = ['x', 'quick']
import tools.batch_check as bc
for B in (8, 32, 64, 128):
    bc.bench("qwen2.5-1.5b", B, 2048)
