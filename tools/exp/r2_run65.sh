timeout 300 python tools/exp/mt_pin.py
