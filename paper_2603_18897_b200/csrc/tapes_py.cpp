// Native payload-tape encoder for Python objects (CPython extension, host).
//
// TapeArena._emit / scalar_bytes (tape.py) restated over the CPython API for
// the exact JSON types -- dict with str keys, list, str, int, float, bool,
// None -- which is what traces hold: mine() over Session objects, the replay
// corpus, predict windows and canonical hashing all encode every event's
// payloads, and the Python encoder costs ~14 us per event.  Semantics are the
// reference's canonical scalar bytes (events.py:94-130): ints as str(int(x)),
// integral floats as str(int(x)) with FLOATSRC, other floats as repr(x),
// strings as UTF-8 (surrogatepass) with the NFC bytes appended when
// unicodedata.normalize("NFC") differs.  A payload holding anything else
// (tuples, subclasses, numpy scalars, non-str keys) is left to the Python
// encoder: encode() reports it and the caller takes the exact slow path for
// that payload, so results never differ.
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

enum { T_NULL = 0, T_FALSE, T_TRUE, T_INT, T_FLOAT, T_STR, T_LIST, T_DICT };
enum { F_NFC = 1, F_FLOATSRC = 2, F_NAN = 4, F_ASCII = 8 };

#pragma pack(push, 1)
struct Node {
  uint8_t type, flags;
  uint16_t pad;
  int32_t key;
  uint32_t a, b;
};
#pragma pack(pop)
static_assert(sizeof(Node) == 16, "tape node");

struct Out {
  std::vector<Node> nodes;
  std::vector<uint8_t> bytes;
  PyObject* objs = nullptr;  // list or NULL (keep_objects)
  PyObject* ids = nullptr;   // KeyTable.ids
  PyObject* names = nullptr; // KeyTable.names
  PyObject* nfc = nullptr;   // unicodedata.normalize
  int64_t byte_base = 0;
};

enum Status { OK = 0, FALLBACK = 1, ERROR = 2 };

void put(Out& o, const char* p, size_t n) { o.bytes.insert(o.bytes.end(), p, p + n); }

Status scalar(Out& o, PyObject* v, int32_t key) {
  Node nd{0, 0, 0, key, (uint32_t)((int64_t)o.bytes.size() - o.byte_base), 0};
  if (v == Py_None) {
    nd.type = T_NULL;
  } else if (v == Py_True) {
    nd.type = T_TRUE;
  } else if (v == Py_False) {
    nd.type = T_FALSE;
  } else if (PyLong_CheckExact(v)) {
    PyObject* s = PyObject_Str(v);
    if (!s) return ERROR;
    Py_ssize_t n;
    const char* c = PyUnicode_AsUTF8AndSize(s, &n);
    if (!c) { Py_DECREF(s); return ERROR; }
    put(o, c, (size_t)n);
    Py_DECREF(s);
    nd.type = T_INT;
    nd.flags = F_ASCII;
    nd.b = (uint32_t)n;
  } else if (PyFloat_CheckExact(v)) {
    const double x = PyFloat_AS_DOUBLE(v);
    if (std::isfinite(x) && x == std::floor(x)) {  // float.is_integer(): str(int(x))
      PyObject* i = PyLong_FromDouble(x);
      if (!i) return ERROR;
      PyObject* s = PyObject_Str(i);
      Py_DECREF(i);
      if (!s) return ERROR;
      Py_ssize_t n;
      const char* c = PyUnicode_AsUTF8AndSize(s, &n);
      if (!c) { Py_DECREF(s); return ERROR; }
      put(o, c, (size_t)n);
      Py_DECREF(s);
      nd.type = T_INT;
      nd.flags = F_FLOATSRC | F_ASCII;
      nd.b = (uint32_t)n;
    } else {  // repr(x): float.__repr__
      char* r = PyOS_double_to_string(x, 'r', 0, Py_DTSF_ADD_DOT_0, nullptr);
      if (!r) return ERROR;
      const size_t n = strlen(r);
      put(o, r, n);
      PyMem_Free(r);
      nd.type = T_FLOAT;
      nd.flags = (uint8_t)((x != x ? F_NAN : 0) | F_ASCII);
      nd.b = (uint32_t)n;
    }
  } else if (PyUnicode_CheckExact(v)) {
    nd.type = T_STR;
    if (PyUnicode_IS_ASCII(v)) {
      Py_ssize_t n;
      const char* c = PyUnicode_AsUTF8AndSize(v, &n);
      if (!c) return ERROR;
      put(o, c, (size_t)n);
      nd.flags = F_ASCII;
      nd.b = (uint32_t)n;
    } else {
      PyObject* raw = PyUnicode_AsEncodedString(v, "utf-8", "surrogatepass");
      if (!raw) return ERROR;
      const size_t rn = (size_t)PyBytes_GET_SIZE(raw);
      put(o, PyBytes_AS_STRING(raw), rn);
      Py_DECREF(raw);
      nd.b = (uint32_t)rn;
      PyObject* n = PyObject_CallFunction(o.nfc, "sO", "NFC", v);
      if (!n) return ERROR;
      const int same = PyUnicode_Compare(n, v);
      if (same == -1 && PyErr_Occurred()) { Py_DECREF(n); return ERROR; }
      if (same != 0) {
        PyObject* nb = PyUnicode_AsEncodedString(n, "utf-8", "surrogatepass");
        Py_DECREF(n);
        if (!nb) return ERROR;
        const uint32_t len = (uint32_t)PyBytes_GET_SIZE(nb);
        put(o, reinterpret_cast<const char*>(&len), 4);  // little endian, as struct "<I"
        put(o, PyBytes_AS_STRING(nb), len);
        Py_DECREF(nb);
        nd.flags = F_NFC;
      } else {
        Py_DECREF(n);
      }
    }
  } else {
    return FALLBACK;
  }
  o.nodes.push_back(nd);
  if (o.objs && PyList_Append(o.objs, v) < 0) return ERROR;
  return OK;
}

int32_t intern(Out& o, PyObject* k) {
  PyObject* id = PyDict_GetItemWithError(o.ids, k);
  if (id) return (int32_t)PyLong_AsLong(id);
  if (PyErr_Occurred()) return -2;
  const Py_ssize_t kid = PyList_GET_SIZE(o.names);
  PyObject* num = PyLong_FromSsize_t(kid);
  if (!num) return -2;
  const int rc = PyDict_SetItem(o.ids, k, num);
  Py_DECREF(num);
  if (rc < 0 || PyList_Append(o.names, k) < 0) return -2;
  return (int32_t)kid;
}

Status emit(Out& o, PyObject* v, int32_t key, int depth) {
  if (depth > 900) return FALLBACK;  // Python's own recursion limit decides
  if (PyDict_CheckExact(v)) {
    const size_t idx = o.nodes.size();
    o.nodes.push_back(Node{T_DICT, 0, 0, key, 0, 0});
    if (o.objs && PyList_Append(o.objs, v) < 0) return ERROR;
    Py_ssize_t pos = 0;
    PyObject *k, *x;
    uint32_t n = 0;
    while (PyDict_Next(v, &pos, &k, &x)) {
      if (!PyUnicode_CheckExact(k)) return FALLBACK;  // non-str keys: the Python path raises
      const int32_t kid = intern(o, k);
      if (kid == -2) return ERROR;
      const Status s = emit(o, x, kid, depth + 1);
      if (s != OK) return s;
      ++n;
    }
    o.nodes[idx].a = n;
    o.nodes[idx].b = (uint32_t)(o.nodes.size() - idx);
    return OK;
  }
  if (PyList_CheckExact(v)) {
    const size_t idx = o.nodes.size();
    o.nodes.push_back(Node{T_LIST, 0, 0, key, 0, 0});
    if (o.objs && PyList_Append(o.objs, v) < 0) return ERROR;
    const Py_ssize_t n = PyList_GET_SIZE(v);
    for (Py_ssize_t i = 0; i < n; ++i) {
      const Status s = emit(o, PyList_GET_ITEM(v, i), -1, depth + 1);
      if (s != OK) return s;
    }
    o.nodes[idx].a = (uint32_t)n;
    o.nodes[idx].b = (uint32_t)(o.nodes.size() - idx);
    return OK;
  }
  return scalar(o, v, key);
}

// encode(payloads, ids, names, node_base, byte_base, objs_or_None)
//   -> (nodes: bytes, data: bytes, refs: list[(node_base, byte_base)])
// Encodes payloads in order and stops before the first one outside the
// native subset (len(refs) tells how many were taken): the caller encodes
// that one with the Python path and calls again on the rest, so the arena is
// byte-identical to encoding every payload in Python.  ids / names / objs
// are updated in place.
PyObject* encode(PyObject*, PyObject* args) {
  PyObject *payloads, *ids, *names, *objs;
  long long node_base0, byte_base0;
  if (!PyArg_ParseTuple(args, "OO!O!LLO", &payloads, &PyDict_Type, &ids, &PyList_Type, &names,
                        &node_base0, &byte_base0, &objs))
    return nullptr;
  PyObject* seq = PySequence_Fast(payloads, "payloads must be a sequence");
  if (!seq) return nullptr;
  static PyObject* nfc = nullptr;
  if (!nfc) {
    PyObject* mod = PyImport_ImportModule("unicodedata");
    if (!mod) { Py_DECREF(seq); return nullptr; }
    nfc = PyObject_GetAttrString(mod, "normalize");
    Py_DECREF(mod);
    if (!nfc) { Py_DECREF(seq); return nullptr; }
  }
  Out o;
  o.ids = ids;
  o.names = names;
  o.nfc = nfc;
  o.objs = objs == Py_None ? nullptr : objs;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyObject* refs = PyList_New(0);
  if (!refs) { Py_DECREF(seq); return nullptr; }
  for (Py_ssize_t i = 0; i < n; ++i) {
    const size_t nodes0 = o.nodes.size(), bytes0 = o.bytes.size();
    const Py_ssize_t objs0 = o.objs ? PyList_GET_SIZE(o.objs) : 0;
    o.byte_base = (int64_t)bytes0;
    const Status s = emit(o, PySequence_Fast_GET_ITEM(seq, i), -1, 0);
    if (s == ERROR) { Py_DECREF(seq); Py_DECREF(refs); return nullptr; }
    if (s == FALLBACK) {  // roll back this payload and stop: the Python encoder takes it
      o.nodes.resize(nodes0);
      o.bytes.resize(bytes0);
      if (o.objs && PyList_SetSlice(o.objs, objs0, PyList_GET_SIZE(o.objs), nullptr) < 0) {
        Py_DECREF(seq); Py_DECREF(refs); return nullptr;
      }
      break;
    }
    PyObject* r = Py_BuildValue("(LL)", (long long)(node_base0 + (long long)nodes0),
                                (long long)(byte_base0 + (long long)bytes0));
    if (!r || PyList_Append(refs, r) < 0) { Py_XDECREF(r); Py_DECREF(seq); Py_DECREF(refs); return nullptr; }
    Py_DECREF(r);
  }
  Py_DECREF(seq);
  PyObject* nb = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(o.nodes.data()),
                                           (Py_ssize_t)(o.nodes.size() * sizeof(Node)));
  PyObject* db = PyBytes_FromStringAndSize(reinterpret_cast<const char*>(o.bytes.data()),
                                           (Py_ssize_t)o.bytes.size());
  if (!nb || !db) { Py_XDECREF(nb); Py_XDECREF(db); Py_DECREF(refs); return nullptr; }
  return Py_BuildValue("(NNN)", nb, db, refs);
}

PyMethodDef methods[] = {
    {"encode", encode, METH_VARARGS, "Encode payloads into tape nodes / bytes (tape.py layout)."},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_tapes", "Native payload-tape encoder.", -1,
                      methods};

}  // namespace

PyMODINIT_FUNC PyInit__tapes(void) { return PyModule_Create(&module); }
