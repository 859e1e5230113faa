LIBS="default w3k4" TLIBS="" bash scripts/gpu/ab_sg.sh
bash scripts/gpu/validate.sh
