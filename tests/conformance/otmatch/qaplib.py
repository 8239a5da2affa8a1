from . import _out_of_scope

load_bundled_instance = _out_of_scope("otmatch.qaplib.load_bundled_instance")
format_qaplib_dat = _out_of_scope("otmatch.qaplib.format_qaplib_dat")
