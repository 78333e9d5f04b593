TAG=default python scripts/step_time.py
TAG=pair FTB_PAIR=1 python scripts/step_time.py
TAG=default2 python scripts/step_time.py
TAG=nointerleave FTB_INTERLEAVE=0 python scripts/step_time.py
