import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from conftest import load_screen_case
from paper_1707_05647_b200 import screen, ScreeningConfig
c = load_screen_case('t4_default')
res = screen(c['image'], c['template'], ScreeningConfig())
print(len(res.candidates), res.stats)
