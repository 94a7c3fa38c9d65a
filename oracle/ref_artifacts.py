"""TEST INFRASTRUCTURE ONLY. Writes the reference's artifacts
(artifacts.cpp:130-143, run_and_write_artifacts) for a JSON config, using
oracle/_ref/libbp_ref.so. Runs without numpy in the process (importing numpy
first crashes the reference's std::filesystem path in this image).
    python oracle/ref_artifacts.py '<config json>' <out_dir>"""
import ctypes
import os
import sys

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libbp_ref.so"))
lib.bpref_write_artifacts.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
lib.bpref_last_error.restype = ctypes.c_char_p
rc = lib.bpref_write_artifacts(sys.argv[1].encode(), sys.argv[2].encode())
if rc:
    sys.exit("reference error: " + lib.bpref_last_error().decode())
